"""C4 bf16 32768^3 A/B of two libgpcx builds: run as two processes alternately
(GPCX_LIB_PATH), 5 timed calls each, TFLOP/s."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_05655_b200 import device as D
s = int(os.environ.get("C4N", "32768"))
A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
ws = D.matmul_workspace(2, s, s, s)
D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); D.matmul(2, A, B, Cm, ws); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(json.dumps({"lib": os.environ.get("GPCX_LIB_PATH", "new"), "ms": round(ms, 2), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1)}))
