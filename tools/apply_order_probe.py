"""C3 LUT_CORRECT (equalize, stretch) step time with L2 flushed between
steps (a 512 MiB write outside the timed events), so only reuse WITHIN a
step counts: the apply pass reading the image back-to-front picks up the
tail the count / min-max pass just left in L2.  CUDA events, median of 9."""
import json, statistics, sys
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
n = 32768 * 32768
img = D.synth_image(0, 0x5EED, 32768, 32768)
out = torch.empty_like(img)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for mode, name in [(0, "equalize"), (1, "stretch")]:
    for flushed in (True, False):
        ts = []
        for i in range(10):
            if flushed:
                flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); D.lut_correct(img, out, mode, lut, stats, ws); b.record(); torch.cuda.synchronize()
            if i: ts.append(a.elapsed_time(b))
        res[f"{name}{'' if flushed else '_noflush'}"] = round(statistics.median(ts), 4)
print(json.dumps(res))
