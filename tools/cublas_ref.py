"""cuBLAS (torch.matmul) bf16 reference timing at the C4 shape and 8192^3,
sustained like tools/c4_ab.py (1 warm-up + 3 timed, CUDA events, NVML
clocks) -- the library baseline our tcgen05 kernel is compared with."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
for s in (8192, 16384, 32768):
    a = torch.randn(s, s, device="cuda").to(torch.bfloat16)
    b = torch.randn(s, s, device="cuda").to(torch.bfloat16)
    torch.matmul(a, b); torch.cuda.synchronize()
    reps = 3 if s == 32768 else 20
    ts = []
    with bench.Clocks(0) as clk:
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); c = torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1)); del c
    ms = statistics.median(ts)
    print(json.dumps({"cublas_bf16": s, "ms": round(ms, 3), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1),
                      "clocks": clk.summary()}), flush=True)
    del a, b
    torch.cuda.empty_cache()
