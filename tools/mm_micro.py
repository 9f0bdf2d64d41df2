"""MATMUL throughput per precision and size on one GPU (CUDA events around
gpcx_matmul_device, i.e. operand prep + GEMM; median of reps).

    python tools/mm_micro.py [--sizes 4096,8192,16384] [--precs f32,tf32,bf16]
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
    ap.add_argument("--sizes", default="4096,8192,16384")
    ap.add_argument("--precs", default="bf16,tf32,f32")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_1505_05655_b200 import device as D
    from paper_1505_05655_b200 import PREC_BY_NAME
    out = {}
    for s in map(int, args.sizes.split(",")):
        A = D.synth_matrix(1, 1, s, s)
        B = D.synth_matrix(1, 2, s, s)
        Cm = torch.empty(s, s, device="cuda")
        for pname in args.precs.split(","):
            if pname == "f32" and s > 8192:
                continue
            prec = PREC_BY_NAME[pname]
            ws = D.matmul_workspace(prec, s, s, s)
            ts = []
            for _ in range(args.reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                D.matmul(prec, A, B, Cm, ws)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts[1:])
            out[f"{pname}/{s}"] = {"ms": round(ms, 3), "TFLOP/s": round(2 * s ** 3 / ms / 1e9, 1)}
            print(pname, s, out[f"{pname}/{s}"], flush=True)
            del ws
        del A, B, Cm
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
