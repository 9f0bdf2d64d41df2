"""Host<->device copy ceilings on this box (pinned host memory, 1 GiB):
H2D alone, D2H alone, both directions concurrently on two streams; run once
per NUMA node when the host has several (taskset to the node's CPUs before
the pinned allocation, so its pages are first-touched there)."""
import json, os, sys, time
import torch

n = 1 << 30
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
h_in.fill_(1); h_out.fill_(2)
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best

h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
dup = timed(both)
print(json.dumps({"cpus": sorted(os.sched_getaffinity(0))[:4], "h2d_GBs": round(n / h2d / 1e9, 1),
                  "d2h_GBs": round(n / d2h / 1e9, 1), "duplex_each_GBs": round(n / dup / 1e9, 1)}))
