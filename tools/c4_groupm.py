"""C4 (32768^3 bf16) sustained A/B over the pair kernel's raster group
height (GPCX_TC_GROUPM), interleaved rounds; CUDA events + NVML clocks."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_05655_b200 import device as D
import bench
s = 32768
A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
ws = D.matmul_workspace(2, s, s, s)
D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
for rnd in range(2):
    for gm in sys.argv[1:]:
        os.environ["GPCX_TC_GROUPM"] = gm
        ts = []
        with bench.Clocks(0) as clk:
            for _ in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); D.matmul(2, A, B, Cm, ws); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(json.dumps({"round": rnd, "group_m": gm, "ms": round(ms, 2), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1),
                          "sm_mhz": clk.summary()["sm_mhz"]}), flush=True)
