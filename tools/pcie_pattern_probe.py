"""The C3 e2e copy pattern without the GPU work: `inflight` host threads,
each looping H2D(2 GiB) -> D2H(2 GiB) on its own stream from pinned
buffers.  Compares with bench's LUT e2e (same pattern + the LUT kernel)."""
import json, sys, threading, time
import torch
n = 2 << 30
inflight = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = 10
bufs = []
for _ in range(inflight):
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    bufs.append((h_in, h_out, d, torch.cuda.Stream()))
def worker(k, count):
    h_in, h_out, d, s = bufs[k]
    with torch.cuda.stream(s):
        for _ in range(count):
            d.copy_(h_in, non_blocking=True)
            h_out.copy_(d, non_blocking=True)
            s.synchronize()
for k in range(inflight):
    worker(k, 1)
t = time.perf_counter()
ts = [threading.Thread(target=worker, args=(k, reps)) for k in range(inflight)]
[x.start() for x in ts]; [x.join() for x in ts]
wall = time.perf_counter() - t
print(json.dumps({"inflight": inflight, "ms_per_request": round(1e3 * wall / (reps * inflight), 2),
                  "GBs_each_way": round(n * reps * inflight / wall / 1e9, 1)}))
