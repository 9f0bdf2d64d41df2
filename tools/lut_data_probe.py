"""Fused LUT_CORRECT (equalize) time at C3 size vs the image's value
distribution: the count pass's smem atomics depend on how many lanes of a
warp hit the same word.  CUDA events, median of 5."""
import json, sys, statistics
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
n = 32768 * 32768
out = torch.empty(n, dtype=torch.int16, device="cuda")
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
g = torch.Generator(device="cuda").manual_seed(1)
imgs = {
    "ramp12": lambda: D.synth_image(0, 0x5EED, 32768, 32768),
    "uniform16": lambda: D.synth_image(1, 0x5EED, 32768, 32768),
    "constant": lambda: torch.full((n,), 1234, dtype=torch.int16, device="cuda"),
    "two_values": lambda: (torch.randint(0, 2, (n,), device="cuda", generator=g, dtype=torch.int16) * 3000 + 100),
    "8bit_scaled": lambda: (torch.randint(0, 256, (n,), device="cuda", generator=g, dtype=torch.int16) * 128),
    "msb12_x16": lambda: (torch.randint(0, 4096, (n,), device="cuda", generator=g, dtype=torch.int16) * 16),
    "msb10_x64": lambda: (torch.randint(0, 1024, (n,), device="cuda", generator=g, dtype=torch.int16) * 64),
    "msb8_x256": lambda: (torch.randint(0, 256, (n,), device="cuda", generator=g, dtype=torch.int32) * 256).to(torch.int16),
    "ramp12_x16": lambda: ((D.synth_image(0, 0x5EED, 32768, 32768).to(torch.int32) - 900) * 16).to(torch.int16),
    "half_flat": lambda: torch.where(torch.arange(n, device="cuda") < n // 2, torch.tensor(500, dtype=torch.int16, device="cuda"),
                                     D.synth_image(0, 0x5EED, 32768, 32768)),
}
res = {}
only = sys.argv[1:]
for name, make in imgs.items():
    if only and name not in only:
        continue
    img = make()
    ts = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); D.lut_correct(img, out, 0, lut, stats, ws); b.record(); torch.cuda.synchronize()
        if i: ts.append(a.elapsed_time(b))
    res[name] = round(statistics.median(ts), 3)
    del img
    torch.cuda.empty_cache()
print(json.dumps(res))
