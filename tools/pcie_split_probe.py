import json, time, torch
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda"); d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best
def split_copy(dst, src, k, off=0):
    c = n // k
    for i in range(k):
        with torch.cuda.stream(streams[off + i]):
            dst[i*c:(i+1)*c].copy_(src[i*c:(i+1)*c], non_blocking=True)
res = {}
for k in (1, 2, 4):
    res[f"h2d_x{k}"] = round(n / timed(lambda: split_copy(d_a, h_in, k)) / 1e9, 1)
    res[f"d2h_x{k}"] = round(n / timed(lambda: split_copy(h_out, d_b, k)) / 1e9, 1)
    res[f"duplex_x{k}"] = round(n / timed(lambda: (split_copy(d_a, h_in, k, 0), split_copy(h_out, d_b, k, 4))) / 1e9, 1)
print(json.dumps(res))
