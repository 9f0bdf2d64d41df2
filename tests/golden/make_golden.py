"""Generates tests/golden/*.json from the numpy restatement (tests/oracle_np.py),
independently of the C oracle it then pins.

    python tests/golden/make_golden.py

The reference (/root/reference) has no LUT / MATMUL code to generate these
from; see oracle/gpcx_oracle.h for the parity status.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_np as NP  # noqa: E402


def lut_cases():
    out = []
    for image, seed, rows, cols in [("ramp12", 0x5EED, 64, 64), ("uniform16", 0x5EED, 64, 64),
                                    ("ramp12", 7, 129, 33), ("uniform16", 99, 1, 1000),
                                    ("ramp12", 0x5EED, 512, 512)]:
        img = NP.image(image, seed, rows, cols)
        for mode in ("equalize", "stretch"):
            lut, st = NP.lut(img, mode)
            probe = sorted({0, 1, st["lo"], st["hi"], (st["lo"] + st["hi"]) // 2, 65535,
                            int(img[0]), int(img[-1])})
            out.append({
                "image": image, "seed": seed, "rows": rows, "cols": cols, "mode": mode,
                "stats": st,
                "out_digest": str(NP.digest(lut[img])),
                "lut_digest": str(NP.digest(lut)),
                "lut_probe": {"at": probe, "values": [int(lut[v]) for v in probe]},
            })
    return out


def matmul_cases():
    out = []
    for seed, m, k, n in [(1, 8, 16, 8), (0x5EED, 33, 70, 17), (5, 128, 256, 64)]:
        A = NP.matrix("exact8", seed, m, k)
        B = NP.matrix("exact8", int(NP.splitmix64(np.uint64(seed))), k, n)
        C = A.astype(np.float64) @ B.astype(np.float64)  # exact: 2^-14 grid, small sums
        rows = [0, m // 2, m - 1]
        cols = [0, n // 3, n - 1]
        out.append({"kind": "exact8", "seed": seed, "m": m, "k": k, "n": n, "rows": rows,
                    "cols": cols, "values": C[np.ix_(rows, cols)].tolist()})
    return out


def main():
    (HERE / "lut_golden.json").write_text(json.dumps({"generator": "tests/oracle_np.py",
                                                       "cases": lut_cases()}, indent=1) + "\n")
    (HERE / "matmul_golden.json").write_text(json.dumps({"generator": "tests/oracle_np.py",
                                                          "cases": matmul_cases()}, indent=1) + "\n")


if __name__ == "__main__":
    main()
