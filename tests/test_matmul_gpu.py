"""MATMUL on the B200 vs the f64 CPU oracle.

Tolerances (stated here as the contract):
  |c - c_ref| <= tol * sum_k |a_ik||b_kj|
  f32  (SIMT, fp32 accumulate)               tol = 1e-5
  tf32 (tcgen05 kind::tf32, RNA-rounded in)  tol = 1e-5 vs the oracle run on
        the same tf32-rounded operands (2e-3 vs the unrounded f32 operands)
  bf16 (tcgen05 kind::f16, RNE-rounded in)   tol = 1e-5 vs the oracle run on
        the same bf16-rounded operands (1.6e-2 vs the unrounded operands)
exact8 operands (k * 2^-7) make every product exact: any accumulation order
gives the same bits while sums stay below 2^24 ulps, so small-k exact8
cases are compared bit-for-bit.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1505_05655_b200 as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = {O.PREC_F32: 1e-5, O.PREC_TF32: 1e-5, O.PREC_BF16: 1e-5}
TOL_UNROUNDED = {O.PREC_F32: 1e-5, O.PREC_TF32: 2e-3, O.PREC_BF16: 1.6e-2}
PREC_NAME = {O.PREC_F32: "f32", O.PREC_TF32: "tf32", O.PREC_BF16: "bf16"}


def _mats(kind, seed, m, k, n):
    A = O.synth_matrix(kind, seed, m, k)
    B = O.synth_matrix(kind, O.seed_b(seed), k, n)
    return A, B


def _check(Cg, A, B, prec, rows=None):
    Ar = O.round_matrix(prec, A) if prec != O.PREC_F32 else A
    Br = O.round_matrix(prec, B) if prec != O.PREC_F32 else B
    Cref, ab = O.matmul_f64(Ar, Br, rows)
    got = Cg if rows is None else Cg[rows]
    err = np.abs(got.astype(np.float64) - Cref)
    bound = TOL[prec] * ab + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    assert np.all(err <= bound), f"prec={PREC_NAME[prec]} worst err/bound={worst:.3g}"
    C0, ab0 = O.matmul_f64(A, B, rows)
    assert np.all(np.abs(got.astype(np.float64) - C0) <= TOL_UNROUNDED[prec] * ab0 + 1e-30)


def _run_device(prec, A, B):
    import torch
    from paper_1505_05655_b200 import device as D
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.full((A.shape[0], B.shape[1]), float("nan"), device="cuda")
    ws = D.matmul_workspace(prec, A.shape[0], B.shape[1], A.shape[1])
    D.matmul(prec, dA, dB, dC, ws)
    return dC.cpu().numpy()


# (256, 384, 512): A^T SIMT kernel; (256, 128, 96): k % 64 != 0 -> row-major-A
# kernel; ragged shapes -> the register-staged kernel
SHAPES = [(128, 128, 16), (256, 384, 512), (256, 128, 96), (1, 1, 1), (3, 5, 7), (129, 130, 131),
          (1000, 17, 300), (64, 1024, 4096)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("kind", [O.MAT_UNIFORM32, O.MAT_EXACT8])
def test_sgemm_within_tolerance(gpu, m, n, k, kind):
    A, B = _mats(kind, 0x5EED, m, k, n)
    _check(_run_device(O.PREC_F32, A, B), A, B, O.PREC_F32)


def test_sgemm_exact8_bit_exact(gpu):
    A, B = _mats(O.MAT_EXACT8, 9, 256, 512, 384)
    Cg = _run_device(O.PREC_F32, A, B)
    Cref, _ = O.matmul_f64(A, B)
    assert np.array_equal(Cg.astype(np.float64), Cref)


def test_sgemm_strided_operands(gpu):
    import torch
    from paper_1505_05655_b200 import device as D
    A, B = _mats(O.MAT_UNIFORM32, 3, 200, 96, 160)
    big_a = torch.zeros(200, 100, device="cuda")
    big_a[:, :96] = torch.from_numpy(A)
    big_b = torch.zeros(96, 170, device="cuda")
    big_b[:, :160] = torch.from_numpy(B)
    big_c = torch.zeros(200, 165, device="cuda")
    D.matmul(O.PREC_F32, big_a[:, :96], big_b[:, :160], big_c[:, :160])
    _check(big_c[:, :160].cpu().numpy(), A, B, O.PREC_F32)
    assert float(big_c[:, 160:].abs().max()) == 0.0


@pytest.mark.parametrize("m,n,k", [(256, 384, 512), (1024, 640, 192)])
def test_sgemm_kernels_agree_bitwise(gpu, monkeypatch, m, n, k):
    """The three SIMT kernels -- A^T (with workspace), row-major A (without),
    register-staged (GPCX_SGEMM=8x2) -- fma-accumulate each output over k in
    ascending order, so they must agree bit for bit."""
    import torch
    from paper_1505_05655_b200 import device as D
    A, B = _mats(O.MAT_UNIFORM32, 21, m, k, n)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ws = D.matmul_workspace(O.PREC_F32, m, n, k)
    assert ws is not None and ws.numel() == m * k * 4
    outs = []
    for variant, w in (("", ws), ("", None), ("8x2", None)):
        monkeypatch.setenv("GPCX_SGEMM", variant)
        dC = torch.full((m, n), float("nan"), device="cuda")
        D.matmul(O.PREC_F32, dA, dB, dC, w)
        outs.append(dC.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    _check(outs[0], A, B, O.PREC_F32)


def test_sgemm_c2_size_sampled(gpu):
    """Config C2 (4096^3, f32) checked on 64 sampled rows."""
    A, B = _mats(O.MAT_UNIFORM32, 0x5EED, 4096, 4096, 4096)
    Cg = _run_device(O.PREC_F32, A, B)
    rows = np.linspace(0, 4095, 64).astype(np.uint64)
    _check(Cg, A, B, O.PREC_F32, rows)


TC = [O.PREC_BF16, O.PREC_TF32]
TC_SHAPES = [(128, 256, 64), (256, 512, 1024), (1, 1, 1), (3, 5, 7), (129, 257, 100), (300, 1000, 520),
             (1024, 768, 4096)]


@pytest.fixture(params=["1sm", "2sm"])
def tc_kernel(request, monkeypatch):
    """Runs a test on the 1-SM (128x256) and the CTA-pair (256x256) kernel."""
    monkeypatch.setenv("GPCX_TC_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("prec", TC)
@pytest.mark.parametrize("m,n,k", TC_SHAPES)
def test_tensor_core_within_tolerance(gpu, tc_kernel, prec, m, n, k):
    A, B = _mats(O.MAT_UNIFORM32, 0x5EED, m, k, n)
    _check(_run_device(prec, A, B), A, B, prec)


@pytest.mark.parametrize("prec", TC)
def test_tensor_core_exact8_bit_exact(gpu, tc_kernel, prec):
    """exact8 operands are exact in bf16 / tf32 and their products are exact
    in fp32; with |partial sums| < 2^24 ulps the result is order-free."""
    A, B = _mats(O.MAT_EXACT8, 11, 384, 512, 768)
    Cg = _run_device(prec, A, B)
    Cref, _ = O.matmul_f64(A, B)
    assert np.array_equal(Cg.astype(np.float64), Cref)


@pytest.mark.parametrize("prec", TC)
def test_tensor_core_kernels_agree_bitwise(gpu, prec, monkeypatch):
    """Same K order per output in both kernels -> identical bits."""
    A, B = _mats(O.MAT_UNIFORM32, 17, 1000, 1500, 700)
    monkeypatch.setenv("GPCX_TC_KERNEL", "1sm")
    c1 = _run_device(prec, A, B)
    monkeypatch.setenv("GPCX_TC_KERNEL", "2sm")
    c2 = _run_device(prec, A, B)
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("prec", TC)
def test_tensor_core_many_tiles_and_strides(gpu, tc_kernel, prec):
    """More output tiles than SMs (persistent loop, both TMEM buffers) and
    strided operands."""
    import torch
    from paper_1505_05655_b200 import device as D
    m, n, k = 2304, 4608, 256  # 18 x 18 = 324 tiles > 148 SMs
    A, B = _mats(O.MAT_UNIFORM32, 13, m, k, n)
    big_a = torch.zeros(m, k + 8, device="cuda")
    big_a[:, :k] = torch.from_numpy(A)
    big_c = torch.full((m, n + 4), -7.0, device="cuda")
    ws = D.matmul_workspace(prec, m, n, k)
    D.matmul(prec, big_a[:, :k], torch.from_numpy(B).cuda(), big_c[:, :n], ws)
    Cg = big_c[:, :n].cpu().numpy()
    rows = np.arange(0, m, 7).astype(np.uint64)
    _check(Cg, A, B, prec, rows)
    assert float(big_c[:, n:].sub(-7.0).abs().max()) == 0.0


@pytest.mark.parametrize("prec,name", [(O.PREC_BF16, "bf16"), (O.PREC_TF32, "tf32")])
def test_gpcx_run_matmul_tensor_core(gpu, prec, name):
    m, k, n = 200, 300, 400
    A, B = _mats(O.MAT_UNIFORM32, 21, m, k, n)
    res, payload = G.run("MATMUL", f"m={m},k={k},n={n},prec={name}", np.concatenate([A.ravel(), B.ravel()]))
    assert res["prec"] == name
    _check(payload.view(np.float32).reshape(m, n), A, B, prec)


def test_gpcx_run_matmul_f32(gpu):
    m, k, n = 70, 90, 110
    A, B = _mats(O.MAT_UNIFORM32, 5, m, k, n)
    res, payload = G.run("MATMUL", f"m={m},k={k},n={n}", np.concatenate([A.ravel(), B.ravel()]))
    assert res == {"m": str(m), "n": str(n), "k": str(k), "prec": "f32"}
    _check(payload.view(np.float32).reshape(m, n), A, B, O.PREC_F32)


@pytest.mark.parametrize("prec,m,k,n", [("f32", 4096, 4096, 4096), ("bf16", 4100, 4097, 4104)])
def test_gpcx_run_matmul_block_rows_invariant(gpu, prec, m, k, n):
    """Block-row sharding (device 0 bound 3x; B staged in k-slices and
    completed by peer copies) gives the bitwise same C."""
    A, B = _mats(O.MAT_UNIFORM32, 6, m, k, n)  # >= 2^36 flop: above the sharding threshold
    payload_in = np.concatenate([A.ravel(), B.ravel()])
    params = f"m={m},k={k},n={n},prec={prec}"
    _, one = G.run("MATMUL", params, payload_in)
    try:
        G.init([0, 0, 0])
        _, three = G.run("MATMUL", params, payload_in)
    finally:
        G.init([0])
    assert np.array_equal(one, three)
    rows = np.arange(0, m, 397)
    C = one.view(np.float32).reshape(m, n)
    _check(C, A, B, O.PREC_F32 if prec == "f32" else O.PREC_BF16, rows=rows)


@pytest.mark.parametrize("prec", TC)
@pytest.mark.parametrize("pad_a,pad_b", [(3, 1), (4, 4), (1, 7)])
def test_tensor_core_operand_prep_strides(gpu, prec, pad_a, pad_b):
    """Operand preparation on row pitches that break (or keep) 16-byte
    alignment, and K / N not multiples of the 8-value chunks or 64-wide
    transpose tiles: the prepared operands (and so C) stay exact."""
    import torch
    from paper_1505_05655_b200 import device as D
    m, k, n = 333, 203, 141
    A, B = _mats(O.MAT_UNIFORM32, 23, m, k, n)
    big_a = torch.zeros(m, k + pad_a, device="cuda")
    big_a[:, :k] = torch.from_numpy(A)
    big_b = torch.zeros(k, n + pad_b, device="cuda")
    big_b[:, :n] = torch.from_numpy(B)
    Cm = torch.empty(m, n, device="cuda")
    D.matmul(prec, big_a[:, :k], big_b[:, :n], Cm, D.matmul_workspace(prec, m, n, k))
    _check(Cm.cpu().numpy(), A, B, prec)


@pytest.mark.slow
@pytest.mark.parametrize("prec", [O.PREC_BF16, O.PREC_TF32])
def test_c4_full_size_sampled(gpu, prec):
    """Config C4 exactly as bench.py runs it (32768^3, prec=bf16 and its
    tf32 variant, operands synthesised on the device): sampled rows spread
    over all of C against the f64 oracle on the same rounded operands."""
    import torch
    from paper_1505_05655_b200 import device as D
    s = 32768
    A = D.synth_matrix(O.MAT_UNIFORM32, 0x5EED, s, s)
    B = D.synth_matrix(O.MAT_UNIFORM32, O.seed_b(0x5EED), s, s)
    Cm = torch.empty(s, s, device="cuda")
    D.matmul(prec, A, B, Cm, D.matmul_workspace(prec, s, s, s))
    rows = np.array([0, 255, 256, 12345, 20000, 32767])
    got = Cm[torch.from_numpy(rows).cuda()].cpu().numpy()
    a_rows = A[torch.from_numpy(rows).cuda()].cpu().numpy()
    del A, Cm
    b = B.cpu().numpy()
    del B
    torch.cuda.empty_cache()
    _check(got, a_rows, b, prec)
