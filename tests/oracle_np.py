"""Second, independent restatement of the LUT / MATMUL task contract in
numpy (vectorised, no loops over pixels), used to cross-check the C oracle
bit-for-bit.  TEST INFRASTRUCTURE.

Formulas: SURVEY.md §8a' (LUT_GEN equalize / stretch), §8d (splitmix64
generators).  Written from the formulas, not from oracle/gpcx_oracle.c.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def image(kind: str, seed: int, rows: int, cols: int) -> np.ndarray:
    r = np.arange(rows, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    h = splitmix64(np.uint64(seed) ^ (r * np.uint64(cols) + c))
    if kind == "uniform16":
        return (h & np.uint64(0xFFFF)).astype(np.uint16).ravel()
    span = max(rows + cols - 2, 1)
    ramp = (3071 * (r + c).astype(np.int64)) // span
    noise = (h >> np.uint64(58)).astype(np.int64) - 32
    return np.clip(1024 + ramp + noise, 0, 65535).astype(np.uint16).ravel()


def matrix(kind: str, seed: int, rows: int, cols: int) -> np.ndarray:
    idx = np.arange(rows * cols, dtype=np.uint64)
    h = splitmix64(np.uint64(seed) ^ idx)
    if kind == "exact8":
        v = (h >> np.uint64(56)).astype(np.uint8).view(np.int8).astype(np.float32) / 128.0
    else:
        v = ((h >> np.uint64(40)).astype(np.float64) / 16777216.0 * 2.0 - 1.0).astype(np.float32)
    return v.reshape(rows, cols)


def lut(img: np.ndarray, mode: str) -> tuple[np.ndarray, dict]:
    hist = np.bincount(img.astype(np.int64), minlength=65536).astype(np.uint64)
    v = np.arange(65536, dtype=np.uint64)
    nz = np.nonzero(hist)[0]
    if nz.size == 0:
        return v.astype(np.uint16), {"n": 0, "lo": 0, "hi": 0, "cdf_min": 0}
    lo, hi = int(nz[0]), int(nz[-1])
    n = int(hist.sum())
    st = {"n": n, "lo": lo, "hi": hi, "cdf_min": int(hist[lo]) if mode == "equalize" else 0}
    if mode == "stretch":
        if hi == lo:
            return v.astype(np.uint16), st
        span = np.uint64(hi - lo)
        mid = ((v - np.uint64(lo)) * np.uint64(65535) + span // np.uint64(2)) // span
        out = np.where(v <= lo, 0, np.where(v >= hi, 65535, mid))
        return out.astype(np.uint16), st
    cdf = np.cumsum(hist, dtype=np.uint64)
    cdf_min = hist[lo]
    d = np.uint64(n) - cdf_min
    if d == 0:
        return v.astype(np.uint16), st
    with np.errstate(over="ignore"):
        val = ((cdf - cdf_min) * np.uint64(65535) + d // np.uint64(2)) // d
    out = np.where(v < lo, 0, val)
    return out.astype(np.uint16), st


def digest(v: np.ndarray, index0: int = 0) -> int:
    i = np.arange(v.size, dtype=np.uint64) + np.uint64(index0)
    h = splitmix64((i << np.uint64(16)) | v.astype(np.uint64))
    with np.errstate(over="ignore"):
        return int(np.sum(h, dtype=np.uint64))


def round_tf32(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    special = (u & np.uint32(0x7F800000)) == np.uint32(0x7F800000)
    r = ((u.astype(np.uint64) + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return np.where(special, u, r).view(np.float32)
