"""Pinning the CPU oracle (oracle/gpcx_oracle.c) before it is trusted.

The reference holds no golden vector for LUT / MATMUL, so
the oracle is pinned by
  * the known-answer tests SURVEY.md §8c lists (hand-computed),
  * an independent numpy restatement (tests/oracle_np.py) that must agree
    bit-for-bit on seeded inputs,
  * the committed golden fixtures (tests/golden/, made by
    tests/golden/make_golden.py) so the oracle cannot drift silently,
  * the reference's own invariance contract: results bitwise independent of
    the worker count (proj/include/gpc/parexec.hpp:11-31).
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import oracle_np as NP
from oracle import oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


# ---------------------------------------------------------------- KATs ---

def test_constant_image_gives_identity_lut():
    img = np.full(64, 1234, dtype=np.uint16)
    for mode in (O.LUT_EQUALIZE, O.LUT_STRETCH):
        lut, st = O.lut_gen(img, mode)
        assert np.array_equal(lut, np.arange(65536, dtype=np.uint16))
        # cdf_min is an equalize statistic; stretch reports 0
        assert st == {"n": 64, "lo": 1234, "hi": 1234, "cdf_min": 64 if mode == O.LUT_EQUALIZE else 0}


@pytest.mark.parametrize("mode", [O.LUT_EQUALIZE, O.LUT_STRETCH])
def test_two_level_image_maps_to_extremes(mode):
    a, b = 300, 40000
    img = np.array([a] * 5 + [b] * 11, dtype=np.uint16)
    lut, st = O.lut_gen(img, mode)
    assert lut[a] == 0 and lut[b] == 65535
    out, _, _ = O.lut_correct(img, mode)
    assert set(out.tolist()) == {0, 65535}
    assert st["lo"] == a and st["hi"] == b


def test_hand_computed_4x4_equalize():
    # values: 10 x4, 20 x4, 30 x4, 40 x4 -> cdf 4,8,12,16; cdf_min=4, D=12
    img = np.array([10, 20, 30, 40] * 4, dtype=np.uint16)
    lut, st = O.lut_gen(img, O.LUT_EQUALIZE)
    # LUT[v] = ((cdf-4)*65535 + 6) // 12
    assert lut[10] == 0
    assert lut[20] == (4 * 65535 + 6) // 12 == 21845
    assert lut[30] == (8 * 65535 + 6) // 12 == 43690
    assert lut[40] == 65535
    assert lut[9] == 0 and lut[15] == 0 and lut[25] == 21845 and lut[65535] == 65535
    assert st == {"n": 16, "lo": 10, "hi": 40, "cdf_min": 4}


def test_hand_computed_stretch_rounding():
    img = np.array([100, 103, 200], dtype=np.uint16)
    lut, _ = O.lut_gen(img, O.LUT_STRETCH)
    # ((v-100)*65535 + 50) // 100, round half up like demosaic.cpp:37-46
    assert lut[103] == (3 * 65535 + 50) // 100 == 1966
    assert lut[150] == (50 * 65535 + 50) // 100 == 32768
    assert lut[100] == 0 and lut[99] == 0 and lut[200] == 65535 and lut[60000] == 65535


def test_identity_lut_apply_is_identity():
    img = O.synth_image(O.IMG_UNIFORM16, 7, 33, 17)
    out = O.lut_apply(np.arange(65536, dtype=np.uint16), img)
    assert np.array_equal(out, img)


def test_matmul_identity_and_permutation_exact():
    rng = np.random.default_rng(1)
    A = rng.integers(-8, 8, size=(9, 13)).astype(np.float32)
    I = np.eye(13, dtype=np.float32)
    C, _ = O.matmul_f64(A, I)
    assert np.array_equal(C, A.astype(np.float64))
    P = np.eye(13, dtype=np.float32)[rng.permutation(13)]
    C, _ = O.matmul_f64(A, P)
    assert np.array_equal(C, A.astype(np.float64) @ P.astype(np.float64))
    assert np.array_equal(O.matmul_f32(A, P), (A.astype(np.float64) @ P).astype(np.float32))


def test_matmul_small_integers_exact_and_absprod():
    A = np.array([[1, -2], [3, 4]], dtype=np.float32)
    B = np.array([[5, 6, -7], [8, 9, 10]], dtype=np.float32)
    C, ab = O.matmul_f64(A, B)
    assert C.tolist() == [[-11, -12, -27], [47, 54, 19]]
    assert ab.tolist() == [[21, 24, 27], [47, 54, 61]]


def test_rounding_kats():
    # tf32: 10 mantissa bits, ties away from zero (cvt.rna.tf32.f32)
    one_plus_half_ulp = np.float32(1.0 + 2.0 ** -11)
    assert O.orc.orc_round_tf32(float(one_plus_half_ulp)) == 1.0 + 2.0 ** -10
    assert O.orc.orc_round_tf32(-float(one_plus_half_ulp)) == -(1.0 + 2.0 ** -10)
    # bf16: 7 mantissa bits, ties to even
    assert O.orc.orc_round_bf16(1.0 + 2.0 ** -8) == 1.0
    assert O.orc.orc_round_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    x = O.synth_matrix(O.MAT_UNIFORM32, 3, 64, 64).ravel() * 1000
    ours = O.round_matrix(O.PREC_BF16, x)
    theirs = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))


def test_tf32_rounding_matches_numpy_restatement():
    x = O.synth_matrix(O.MAT_UNIFORM32, 4, 32, 32).ravel()
    assert np.array_equal(O.round_matrix(O.PREC_TF32, x).view(np.uint32),
                          NP.round_tf32(x).view(np.uint32))


# ------------------------------------------- independent restatement ---

@pytest.mark.parametrize("kind,name", [(O.IMG_RAMP12, "ramp12"), (O.IMG_UNIFORM16, "uniform16")])
@pytest.mark.parametrize("rows,cols", [(1, 1), (2, 3), (37, 53), (256, 128)])
def test_synth_image_matches_numpy(kind, name, rows, cols):
    assert np.array_equal(O.synth_image(kind, 0x5EED, rows, cols), NP.image(name, 0x5EED, rows, cols))


def test_synth_image_row_band_is_a_slice():
    full = O.synth_image(O.IMG_RAMP12, 9, 40, 24)
    band = O.synth_image(O.IMG_RAMP12, 9, 40, 24, row0=13, nrows=11)
    assert np.array_equal(band, full[13 * 24:24 * 24])


@pytest.mark.parametrize("kind,name", [(O.MAT_EXACT8, "exact8"), (O.MAT_UNIFORM32, "uniform32")])
def test_synth_matrix_matches_numpy(kind, name):
    a = O.synth_matrix(kind, 0x5EED, 31, 47)
    b = NP.matrix(name, 0x5EED, 31, 47)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    if name == "exact8":
        assert np.all(a * 128 == np.round(a * 128)) and a.min() >= -1 and a.max() < 1


@pytest.mark.parametrize("name,kind", [("ramp12", O.IMG_RAMP12), ("uniform16", O.IMG_UNIFORM16)])
@pytest.mark.parametrize("mode,mname", [(O.LUT_EQUALIZE, "equalize"), (O.LUT_STRETCH, "stretch")])
def test_lut_matches_numpy(name, kind, mode, mname):
    img = O.synth_image(kind, 0x5EED, 300, 211)
    lut, st = O.lut_gen(img, mode)
    lut2, st2 = NP.lut(img, mname)
    assert np.array_equal(lut, lut2)
    assert st == st2
    out, lut3, st3 = O.lut_correct(img, mode)
    assert np.array_equal(out, lut2[img])
    assert np.array_equal(lut3, lut2) and st3 == st2


def test_lut_monotone_and_bounded():
    img = O.synth_image(O.IMG_RAMP12, 11, 128, 128)
    for mode in (O.LUT_EQUALIZE, O.LUT_STRETCH):
        lut, st = O.lut_gen(img, mode)
        assert np.all(np.diff(lut.astype(np.int64)) >= 0)
        assert lut[st["hi"]] == 65535


def test_digest_matches_numpy_and_is_order_keyed():
    v = O.synth_image(O.IMG_UNIFORM16, 3, 10, 100)
    assert O.digest_u16(v) == NP.digest(v)
    assert O.digest_u16(v[500:], 500) + O.digest_u16(v[:500], 0) & (2 ** 64 - 1) == O.digest_u16(v)
    w = v.copy()
    w[[3, 4]] = w[[4, 3]]
    if v[3] != v[4]:
        assert O.digest_u16(w) != O.digest_u16(v)


def test_matmul_f64_matches_numpy_float64():
    A = O.synth_matrix(O.MAT_UNIFORM32, 1, 23, 41)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(1), 41, 19)
    C, ab = O.matmul_f64(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.allclose(C, ref, rtol=0, atol=1e-12)
    assert np.allclose(ab, np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64), atol=1e-12)
    rows = np.array([22, 0, 7], dtype=np.uint64)
    Cs, _ = O.matmul_f64(A, B, rows)
    assert np.array_equal(Cs, C[[22, 0, 7]])


# ------------------------------------------------ worker invariance ---

def test_results_independent_of_thread_count():
    img = O.synth_image(O.IMG_UNIFORM16, 5, 512, 300)
    base = O.lut_correct(img, O.LUT_EQUALIZE, threads=1)
    for t in (2, 3, 8):
        out = O.lut_correct(img, O.LUT_EQUALIZE, threads=t)
        assert np.array_equal(out[0], base[0]) and out[2] == base[2]
    A = O.synth_matrix(O.MAT_UNIFORM32, 1, 17, 33)
    B = O.synth_matrix(O.MAT_UNIFORM32, 2, 33, 29)
    c1 = O.matmul_f32(A, B, threads=1)
    for t in (2, 5):
        assert np.array_equal(O.matmul_f32(A, B, threads=t), c1)


# ----------------------------------------------------- golden fixtures ---

def test_golden_fixtures():
    data = json.loads((GOLDEN / "lut_golden.json").read_text())
    for case in data["cases"]:
        kind = {"ramp12": O.IMG_RAMP12, "uniform16": O.IMG_UNIFORM16}[case["image"]]
        mode = {"equalize": O.LUT_EQUALIZE, "stretch": O.LUT_STRETCH}[case["mode"]]
        img = O.synth_image(kind, case["seed"], case["rows"], case["cols"])
        out, lut, st = O.lut_correct(img, mode)
        assert st == case["stats"], case
        assert O.digest_u16(out) == int(case["out_digest"]), case
        assert O.digest_u16(lut) == int(case["lut_digest"]), case
        probe = case["lut_probe"]
        assert [int(lut[v]) for v in probe["at"]] == probe["values"]
    mm = json.loads((GOLDEN / "matmul_golden.json").read_text())
    for case in mm["cases"]:
        kind = {"exact8": O.MAT_EXACT8, "uniform32": O.MAT_UNIFORM32}[case["kind"]]
        A = O.synth_matrix(kind, case["seed"], case["m"], case["k"])
        B = O.synth_matrix(kind, O.seed_b(case["seed"]), case["k"], case["n"])
        C, _ = O.matmul_f64(A, B, np.array(case["rows"], dtype=np.uint64))
        got = C[:, case["cols"]]
        assert np.array_equal(got, np.array(case["values"], dtype=np.float64)), case
