"""Short, deterministic workload for ncu captures (one launch of each hot
kernel at the bench configuration):
  LUT_CORRECT equalize on the C3 scene (32768^2 u16): hist, merge, from_hist, apply
  MATMUL bf16 8192^3 (and tf32 4096^3) through the tcgen05 path
    ncu --set full -k regex:'hist_kernel|apply_kernel|gemm_kernel' ... python tools/prof_target.py
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="lut,mm")
    ap.add_argument("--mm", type=int, default=8192)
    args = ap.parse_args()
    import torch
    from paper_1505_05655_b200 import device as D
    if "c1" in args.what:  # config C1: one 4096^2 LUT_CORRECT (fused_kernel)
        img = D.synth_image(0, 0x5EED, 4096, 4096)
        out = torch.empty_like(img)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
        D.lut_correct(img, out, 0, lut, stats, ws)
        torch.cuda.synchronize()
        del img, out
    if "lut" in args.what:
        n = 32768 * 32768
        img = D.synth_image(0, 0x5EED, 32768, 32768)
        out = torch.empty_like(img)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
        D.lut_correct(img, out, 0, lut, stats, ws)
        D.lut_apply(lut, img, out)  # LUT_APPLY's kernel on the same scene
        torch.cuda.synchronize()
        del img, out
    if "stretch" in args.what:  # C3 scene, mode=stretch: minmax + from_minmax + apply
        n = 32768 * 32768
        img = D.synth_image(0, 0x5EED, 32768, 32768)
        out = torch.empty_like(img)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
        D.lut_correct(img, out, 1, lut, stats, ws)
        torch.cuda.synchronize()
        del img, out
    if "sgemm" in args.what:  # config C2: FP32 SIMT 4096^3
        A = D.synth_matrix(1, 1, 4096, 4096)
        B = D.synth_matrix(1, 2, 4096, 4096)
        Cm = torch.empty(4096, 4096, device="cuda")
        D.matmul(0, A, B, Cm, D.matmul_workspace(0, 4096, 4096, 4096))
        torch.cuda.synchronize()
    if "demosaic" in args.what:  # BAYER_BILINEAR / BAYER_GRADIENT at 16384^2
        img = D.synth_image(1, 3, 16384, 16384)
        for grad in (False, True):
            D.demosaic(grad, 0, img, 16384, 16384)
        torch.cuda.synchronize()
    if "c4" in args.what.split(","):  # config C4: one 32768^3 bf16 MATMUL
        A = D.synth_matrix(1, 1, 32768, 32768)
        B = D.synth_matrix(1, 2, 32768, 32768)
        Cm = torch.empty(32768, 32768, device="cuda")
        ws = D.matmul_workspace(2, 32768, 32768, 32768)
        D.matmul(2, A, B, Cm, ws)
        torch.cuda.synchronize()
        print("done")
        return
    if args.what == "longk2":  # one long-K GEMM with the caller's GPCX_TC_* environment
        A = D.synth_matrix(1, 1, 8192, 32768)
        B = D.synth_matrix(1, 2, 32768, 8192)
        Cm = torch.empty(8192, 8192, device="cuda")
        ws = D.matmul_workspace(2, 8192, 8192, 32768)
        D.matmul(2, A, B, Cm, ws)
        torch.cuda.synchronize()
        print("done")
        return
    if "longk" in args.what:  # C4-like long K, cheaper to replay than 32768^3
        import os
        m = n = 8192
        k = 32768
        A = D.synth_matrix(1, 1, m, k)
        B = D.synth_matrix(1, 2, k, n)
        Cm = torch.empty(m, n, device="cuda")
        ws = D.matmul_workspace(2, m, n, k)
        for kern in ("1sm", "2sm"):
            os.environ["GPCX_TC_KERNEL"] = kern
            D.matmul(2, A, B, Cm, ws)
            torch.cuda.synchronize()
        print("done")
        return
    if "mm" in args.what.split(","):
        s = args.mm
        A = D.synth_matrix(1, 1, s, s)
        B = D.synth_matrix(1, 2, s, s)
        Cm = torch.empty(s, s, device="cuda")
        for prec in (2, 1):
            ws = D.matmul_workspace(prec, s, s, s)
            D.matmul(prec, A, B, Cm, ws)
            torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
