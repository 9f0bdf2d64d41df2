"""C4 (32768^3 bf16) under the power cap: raster group height x ring depth,
interleaved in one process (GPCX_TC_GROUPM / GPCX_TC_STAGES2 are read per
call); reports ms, median SM clock and ms x MHz (SM cycles, which factors
out the box's power / thermal state)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_05655_b200 import device as D
import bench
s = int(os.environ.get("C4N", "32768"))
A = D.synth_matrix(1, 1, s, s); B = D.synth_matrix(1, 2, s, s); Cm = torch.empty(s, s, device="cuda")
ws = D.matmul_workspace(2, s, s, s)
cfgs = [c.split(":") for c in (sys.argv[1:] or ["8:4", "4:4", "16:4", "8:3", "8:5", "2:4"])]
for rep in range(2):
    for gm, st in cfgs:
        os.environ["GPCX_TC_GROUPM"], os.environ["GPCX_TC_STAGES2"] = gm, st
        D.matmul(2, A, B, Cm, ws); torch.cuda.synchronize()
        ts = []
        with bench.Clocks(0) as clk:
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); D.matmul(2, A, B, Cm, ws); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        ms = statistics.median(ts); c = clk.summary()
        print(json.dumps({"group_m": gm, "stages": st, "ms": round(ms, 2), "TFLOP/s": round(2 * s**3 / ms / 1e9, 1),
                          "sm_mhz": c["sm_mhz"], "Mcycles": round(ms * c["sm_mhz"] / 1e3, 1)}), flush=True)
