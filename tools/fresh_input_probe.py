"""Is the fused LUT kernel slower right after its input arrived by H2D DMA?
Events around the kernel on one stream, no other work on the GPU."""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
n = 32768 * 32768
h = D.synth_image(0, 0x5EED, 32768, 32768).cpu().pin_memory()
d_in = torch.empty(n, dtype=torch.int16, device="cuda"); other = torch.empty_like(d_in)
out = torch.empty_like(d_in)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
s = torch.cuda.current_stream()
def run(kind, fn):
    res = []
    for _ in range(3):
        if kind == "h2d_same":
            d_in.copy_(h, non_blocking=True)
        elif kind == "h2d_other":
            other.copy_(h, non_blocking=True)
        elif kind == "d2d_same":
            d_in.copy_(other)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        res.append(round(a.elapsed_time(b), 3))
    return res
other.copy_(h)
fused = lambda: D.lut_correct(d_in, out, 0, lut, stats, ws)
apply = lambda: D.lut_apply(lut, d_in, out)
stretch = lambda: D.lut_correct(d_in, out, 1, lut, stats, ws)
for kind in ("none", "h2d_same", "h2d_other", "d2d_same"):
    print(json.dumps({"before": kind, "fused": run(kind, fused), "apply": run(kind, apply),
                      "stretch": run(kind, stretch)}), flush=True)
