"""Randomised MATMUL parity: random shapes (ragged and aligned, skinny and
square, k from 1 to a few thousand), every precision, through the task-level
C ABI (host buffers, the executor's kernel choice) -- against the f64 oracle
at the stated tolerances (tests/test_matmul_gpu.py)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1505_05655_b200 as G
from oracle import oracle as O
from test_matmul_gpu import PREC_NAME, _check

pytestmark = pytest.mark.gpu


def _shape(rng):
    pick = rng.integers(0, 4)
    if pick == 0:   # small / ragged
        return tuple(int(x) for x in rng.integers(1, 300, 3))
    if pick == 1:   # aligned to the tensor tiles
        return tuple(int(x) * 128 for x in rng.integers(1, 12, 3))
    if pick == 2:   # skinny
        return int(rng.integers(1, 40)), int(rng.integers(500, 3000)), int(rng.integers(1, 2000))
    return tuple(int(x) for x in rng.integers(300, 1600, 3))


# 16 cases by default; GPCX_MM_RANDOM_CASES=60 was run once (60 passed)
@pytest.mark.parametrize("seed", range(int(os.environ.get("GPCX_MM_RANDOM_CASES", "16"))))
def test_matmul_random_shapes(gpu, seed):
    rng = np.random.default_rng(1000 + seed)
    m, k, n = _shape(rng)
    prec = [O.PREC_F32, O.PREC_TF32, O.PREC_BF16][seed % 3]
    kind = O.MAT_UNIFORM32 if rng.random() < 0.7 else O.MAT_EXACT8
    A = O.synth_matrix(kind, seed, m, k)
    B = O.synth_matrix(kind, O.seed_b(seed), k, n)
    _, c = G.run("MATMUL", f"m={m},k={k},n={n},prec={PREC_NAME[prec]}",
                 np.concatenate([A.ravel(), B.ravel()]))
    C = c.view(np.float32).reshape(m, n)
    rows = None if m <= 512 else np.arange(0, m, 7, dtype=np.uint64)
    _check(C, A, B, prec, rows)
