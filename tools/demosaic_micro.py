"""BAYER_* kernel throughput (CUDA events, median of reps): 2 B in + 6 B out
per pixel, HBM-bound.

    python tools/demosaic_micro.py [--sizes 2048,4096,16384]
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
    ap.add_argument("--sizes", default="2048,4096,16384")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_1505_05655_b200 import device as D
    res = {}
    for s in map(int, args.sizes.split(",")):
        img = D.synth_image(1, 7, s, s)
        out = torch.empty(3 * s * s, dtype=torch.int16, device="cuda")
        for grad in (False, True):
            ts = []
            for _ in range(args.reps + 2):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                D.demosaic(grad, 0, img, s, s, out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts[2:])
            res[f"{'gradient' if grad else 'bilinear'}/{s}"] = {
                "ms": round(ms, 4), "Gpx/s": round(s * s / ms / 1e6, 1),
                "GB/s": round(8 * s * s / ms / 1e6, 1)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
