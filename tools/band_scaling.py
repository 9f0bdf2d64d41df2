"""Per-rank work of the N-GPU configs, timed on one B200: what each rank's
kernel costs at band size 1/N (C3 LUT_CORRECT row bands, C4 block rows of
A / C).  Only N=1 is measurable as a whole on this single-GPU pool; this
shows how the sharded compute itself scales (the exchange / replication
steps come on top: the histogram rendezvous is a few microseconds of
system-scope flags, B's all-gather runs under the previous GEMM).

    python tools/band_scaling.py > profiles/r2/band_scaling.txt
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def timed(fn, reps: int, warmup: int = 3) -> float:
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main() -> None:
    import torch
    from paper_1505_05655_b200 import device as D
    rows = cols = 32768
    print("# C3 LUT_CORRECT (equalize, ramp12), one rank's row band on one B200 (fused_kernel, single launch)")
    print("N  band_rows  ms_per_step  Gpx/s_band  x_vs_N1  ideal")
    t1 = None
    for n in (1, 2, 4, 8):
        nr = rows // n
        img = D.synth_image(0, 0x5EED, rows, cols, 0, nr)
        out = torch.empty_like(img)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
        ms = timed(lambda: D.lut_correct(img, out, 0, lut, stats, ws), 20)
        t1 = t1 or ms
        print(f"{n}  {nr:9d}  {ms:11.4f}  {nr * cols / ms / 1e6:10.1f}  {t1 / ms:7.2f}  {n:5d}")
        del img, out
    torch.cuda.empty_cache()
    print("# C4 MATMUL bf16 32768^3, one rank's block rows (m = 32768/N, full n, k; incl. operand prep)")
    print("N  rows  ms_per_step  TFLOP/s_rank  x_vs_N1  ideal")
    t1 = None
    B = D.synth_matrix(1, 7, 32768, 32768)
    for n in (1, 2, 4, 8):
        m = 32768 // n
        A = D.synth_matrix(1, 0x5EED, 32768, 32768, 0, m)
        C = torch.empty(m, 32768, device="cuda")
        ws = D.matmul_workspace(2, m, 32768, 32768)
        ms = timed(lambda: D.matmul(2, A, B, C, ws), 3 if n == 1 else 5, warmup=1)
        t1 = t1 or ms
        print(f"{n}  {m:5d}  {ms:11.3f}  {2.0 * m * 32768 * 32768 / ms / 1e9:12.1f}  {t1 / ms:7.2f}  {n:5d}")
        del A, C, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
