"""MATMUL anchored on values the REFERENCE computes.

The reference has no matrix multiply task, but its polynomial fit builds
the normal equations with two real contractions (gpc::lsq::
build_normal_system, proj/src/lsq.cpp:69-90): A = V^T V, the Hankel matrix
of power sums, and b = V^T y, with V[i][j] = x_i^j.  Both are MATMULs of
the task's convention (row-major A (m x k) times B (k x n)).  With dyadic
abscissae x = k/64 every V entry and every partial sum is exact in f64, so
the oracle's f64 MATMUL must reproduce the reference's numbers bit for
bit, whatever the summation order -- this pins the oracle's MATMUL (layout,
orientation, accumulation) on the reference's own arithmetic.  The B200
MATMUL is then held to the task's stated bars against those same
reference-computed values (f32: 1e-5 * sum|a||b|; tf32 / bf16 against the
unrounded operands: 2e-3 / 1.6e-2), except that for f32 at long k the bar
is the recursive-summation bound gamma_k = k * 2^-24 when that is larger:
power sums are same-sign, so nothing cancels, and the SIMT kernel (like
cuBLAS SGEMM) accumulates each output sequentially over k -- at k = 70000
it is 3.7e-4 * sum|a||b| off.  C2's random-sign operands
(k = 4096) stay within 1e-5."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O


def _system(order: int, n: int, seed: int):
    rng = np.random.default_rng(seed)
    xs = rng.integers(-64, 65, n) / 64.0   # x^j exact in f32 for j <= 3 (<= 21 bits)
    ys = rng.integers(-64, 65, n) / 64.0
    V = np.stack([xs ** j for j in range(order + 1)], axis=1)  # n x (order+1)
    return xs, ys, V


@pytest.mark.parametrize("order,n", [(0, 1), (1, 7), (3, 4097), (3, 12_345)])
def test_oracle_matmul_equals_reference_normal_equations(refl, order, n):
    """n > 4096 crosses the reference's fixed reduction chunk (parexec)."""
    xs, ys, V = _system(order, n, 10 + order)
    a_ref, b_ref = refl.ref_normal_system(xs, ys, order)
    Vt = np.ascontiguousarray(V.T.astype(np.float32))
    a, _ = O.matmul_f64(Vt, V.astype(np.float32))
    b, _ = O.matmul_f64(Vt, ys.astype(np.float32).reshape(n, 1))
    assert np.array_equal(a, a_ref)
    assert np.array_equal(b.ravel(), b_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("prec,tol", [(O.PREC_F32, 1e-5), (O.PREC_TF32, 2e-3), (O.PREC_BF16, 1.6e-2)])
@pytest.mark.parametrize("order,n", [(3, 12_345), (2, 70_000), (3, 1000)])
def test_b200_matmul_vs_reference_normal_equations(gpu, refl, prec, tol, order, n):
    import paper_1505_05655_b200 as G
    name = {O.PREC_F32: "f32", O.PREC_TF32: "tf32", O.PREC_BF16: "bf16"}[prec]
    xs, ys, V = _system(order, n, 20 + order)
    a_ref, b_ref = refl.ref_normal_system(xs, ys, order)
    m1 = order + 1
    Vt = np.ascontiguousarray(V.T.astype(np.float32))
    Vf = np.ascontiguousarray(V.astype(np.float32))
    _, ab = O.matmul_f64(Vt, Vf)  # sum |a||b| per entry
    if prec == O.PREC_F32:
        tol = max(tol, n * 2.0 ** -24)  # gamma_k for same-sign sums
    _, c = G.run("MATMUL", f"m={m1},k={n},n={m1},prec={name}",
                 np.concatenate([Vt.ravel(), Vf.ravel()]))
    C = c.view(np.float32).reshape(m1, m1).astype(np.float64)
    assert np.all(np.abs(C - a_ref) <= tol * ab), (name, np.abs(C - a_ref).max())
    yf = ys.astype(np.float32).reshape(n, 1)
    _, abb = O.matmul_f64(Vt, yf)
    _, c = G.run("MATMUL", f"m={m1},k={n},n=1,prec={name}", np.concatenate([Vt.ravel(), yf.ravel()]))
    got = c.view(np.float32).astype(np.float64)
    assert np.all(np.abs(got - b_ref) <= tol * abb.ravel()), (name, np.abs(got - b_ref).max())
