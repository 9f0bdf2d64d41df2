"""Per-kernel timings of the LUT path on one GPU (CUDA events, median of
reps) for both synthetic images -- the optimisation loop's measurement.

    python tools/lut_micro.py [--rows 32768] [--cols 32768] [--reps 10]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--cols", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--flush", action="store_true",
                    help="write 512 MiB between reps so every rep starts with a cold L2")
    args = ap.parse_args()
    import torch
    from paper_1505_05655_b200 import device as D

    n = args.rows * args.cols
    hist = torch.zeros(65536, dtype=torch.int32, device="cuda")
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    res = {}
    for kind, name in ((0, "ramp12"), (1, "uniform16")):
        img = D.synth_image(kind, 0x5EED, args.rows, args.cols)
        D.lut_hist(img, hist, ws)
        D.lut_from_hist(hist, 0, lut, stats, ws)
        ops = {
            "hist+merge": lambda: D.lut_hist(img, hist, ws),
            "from_hist": lambda: D.lut_from_hist(hist, 0, lut, stats, ws),
            "gen(hist+fused build)": lambda: D.lut_gen(img, 0, lut, stats, ws),
            "correct(fused)": lambda: D.lut_correct(img, out, 0, lut, stats, ws),
            "gen+apply(2 launches)": lambda: (D.lut_gen(img, 0, lut, stats, ws),
                                              D.lut_apply(lut, img, out)),
            "minmax": lambda: D.lut_minmax(img, stats, ws),
            "apply": lambda: D.lut_apply(lut, img, out),
            "copy(torch)": lambda: out.copy_(img),
        }
        bytes_per = {"hist+merge": 2 * n, "from_hist": 0, "minmax": 2 * n, "apply": 4 * n,
                     "copy(torch)": 4 * n, "gen(hist+fused build)": 2 * n,
                     "correct(fused)": 6 * n, "gen+apply(2 launches)": 6 * n}
        for op, fn in ops.items():
            ts = []
            for i in range(args.reps + 2):
                if flush is not None:
                    flush.fill_(i & 0xFF)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts[2:])
            res[f"{name}/{op}"] = {"ms": round(ms, 4),
                                   "GB/s": round(bytes_per[op] / ms / 1e6, 1) if bytes_per[op] else None}
        del img
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
