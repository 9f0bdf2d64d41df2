import sys, statistics, json
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
res = {}
for rows, cols in [(4096, 4096), (1024, 1024), (7, 13)]:
    img = D.synth_image(0, 7, rows, cols); out = torch.empty_like(img)
    lut, st, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
    ts = []
    for i in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); D.lut_correct(img, out, 1, lut, st, ws); b.record(); torch.cuda.synchronize()
        if i > 5: ts.append(a.elapsed_time(b) * 1000)
    res[f"{rows}x{cols}_us"] = round(statistics.median(ts), 1)
print(json.dumps(res))
