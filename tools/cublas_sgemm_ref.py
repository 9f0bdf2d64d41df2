"""cuBLAS FP32 (no TF32) SGEMM at C2 (4096^3) -- the library baseline for
the SIMT reference-precision kernel (L2 flushed between reps like bench.py)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
s = 4096
a = torch.rand(s, s, device="cuda"); b = torch.rand(s, s, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(15):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(json.dumps({"cublas_sgemm_f32": s, "ms": round(ms, 3), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1)}))
