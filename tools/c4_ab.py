"""A/B of the tensor-core kernels on config C4 (32768^3 bf16), sustained:
3 timed calls after 1 warm-up, CUDA events, clocks via NVML."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_05655_b200 import device as D
import bench
s = int(os.environ.get("C4N", "32768"))
A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
ws = D.matmul_workspace(2, s, s, s)
for kern in sys.argv[1:]:
    os.environ["GPCX_TC_KERNEL"] = kern
    D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
    ts = []
    with bench.Clocks(0) as clk:
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); D.matmul(2, A, B, Cm, ws); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(json.dumps({"kernel": kern, "ms": round(ms, 2), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1), "clocks": clk.summary()}), flush=True)
