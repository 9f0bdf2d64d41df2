"""Does the cooperative LUT kernel slow down (or start late) while another
stream is copying over PCIe?  Events around the kernel on its own stream."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
n = 32768 * 32768
img = D.synth_image(0, 0x5EED, 32768, 32768); out = torch.empty_like(img)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
h = torch.empty(2 << 30, dtype=torch.uint8).pin_memory(); d = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
s_copy, s_k = torch.cuda.Stream(), torch.cuda.Stream()
def kernel_ms(with_copy, apply_only=False):
    torch.cuda.synchronize()
    if with_copy == "h2d":
        with torch.cuda.stream(s_copy):
            d.copy_(h, non_blocking=True)
        time.sleep(0.005)
    elif with_copy:
        with torch.cuda.stream(s_copy):
            h.copy_(d, non_blocking=True)
        time.sleep(0.005)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record(s_k)
    if apply_only:
        D.lut_apply(lut, img, out, s_k)
    else:
        D.lut_correct(img, out, 0, lut, stats, ws, s_k)
    b.record(s_k)
    host_us = (time.perf_counter() - t) * 1e6
    torch.cuda.synchronize()
    return round(a.elapsed_time(b), 3), round(host_us, 1)
for i in range(3):
    print(json.dumps({"fused_alone": kernel_ms(False), "fused_with_h2d": kernel_ms("h2d"),
                      "fused_with_d2h": kernel_ms("d2h"),
                      "apply_alone": kernel_ms(False, True), "apply_with_h2d": kernel_ms("h2d", True),
                      "apply_with_d2h": kernel_ms("d2h", True)}), flush=True)
