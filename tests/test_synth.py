"""Header-only synthetic requests (SURVEY.md §8d option ii): synth= /
seed= / samples= make LUT_GEN / LUT_CORRECT / MATMUL generate their inputs
on the GPUs, so the over-cap configs C3 (2 GiB scene) and C4 (32768^3) run
through the served path.  LUT_CORRECT answers the corrected image's
position-keyed digest, MATMUL seeded samples of C -- both checked against
the oracle on the same counter-based inputs."""
from __future__ import annotations

import struct

import numpy as np
import pytest

import paper_1505_05655_b200 as G
from oracle import oracle as O

SEED = 0x5EED


def test_synth_sizing_without_payload():
    big = "rows=32768,cols=32768,synth=ramp12"
    assert G.payload_len("LUT_CORRECT", big) == 0
    assert G.output_len("LUT_CORRECT", big) == 8
    assert G.payload_len("LUT_GEN", big) == 0 and G.output_len("LUT_GEN", big) == 131072
    mm = "m=32768,k=32768,n=32768,prec=bf16,synth=uniform32"
    assert G.payload_len("MATMUL", mm) == 0
    assert G.output_len("MATMUL", mm) == 4096 * 12
    assert G.output_len("MATMUL", mm + ",samples=10") == 120
    # without synth the same dims exceed the 1 GiB wire cap (the reference's rule)
    with pytest.raises(G.GpcxError) as e:
        G.payload_len("LUT_CORRECT", "rows=32768,cols=32768")
    assert e.value.code == "Overflow"


@pytest.mark.parametrize("flag,params,code", [
    ("LUT_CORRECT", "rows=4,cols=4,synth=gauss", "BadValue"),
    ("LUT_CORRECT", "rows=4,cols=4,synth=exact8", "BadValue"),
    ("LUT_APPLY", "rows=4,cols=4,synth=ramp12", "BadValue"),
    ("LUT_CORRECT", "rows=65536,cols=65536,synth=ramp12", "Overflow"),
    ("LUT_CORRECT", "rows=0,cols=4,synth=ramp12", "BadValue"),
    ("MATMUL", "m=4,k=4,n=4,synth=ramp12", "BadValue"),
    ("MATMUL", "m=4,k=4,n=4,synth=exact8,samples=0", "BadValue"),
    ("MATMUL", "m=4,k=4,n=4,synth=exact8,samples=2000000", "BadValue"),
    ("MATMUL", "m=65536,k=65536,n=4,synth=exact8", "Overflow"),
])
def test_synth_rejections(flag, params, code):
    with pytest.raises(G.GpcxError) as e:
        G.payload_len(flag, params)
    assert e.value.code == code


def _samples(blob: bytes):
    return [struct.unpack_from("<IIf", blob, 12 * j) for j in range(len(blob) // 12)]


def _check_samples(samples, kind, seed, m, k, n, prec, tol=1e-5):
    A = O.synth_matrix(kind, seed, m, k)
    B = O.synth_matrix(kind, O.seed_b(seed), k, n)
    if prec != O.PREC_F32:
        A, B = O.round_matrix(prec, A), O.round_matrix(prec, B)
    for j, (r, c, v) in enumerate(samples):
        h_r = O.splitmix64(seed ^ (2 * j)) % m
        h_c = O.splitmix64(seed ^ (2 * j + 1)) % n
        assert (r, c) == (h_r, h_c), j
        a, b = A[r].astype(np.float64), B[:, c].astype(np.float64)
        assert abs(v - float(a @ b)) <= tol * float(np.abs(a) @ np.abs(b)) + 1e-30, (j, r, c)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,mode", [("ramp12", "equalize"), ("uniform16", "stretch")])
@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_synth_lut_correct_digest_and_gen(gpu, kind, mode, devices):
    rows, cols = 4099, 4097  # > 2^24 px: the planner shards over 2 bound devices
    k = O.IMG_RAMP12 if kind == "ramp12" else O.IMG_UNIFORM16
    m = O.LUT_EQUALIZE if mode == "equalize" else O.LUT_STRETCH
    img = O.synth_image(k, 77, rows, cols)
    r_out, r_lut, r_st = O.lut_correct(img, m)
    try:
        G.init(devices)
        params, out = G.run("LUT_CORRECT", f"rows={rows},cols={cols},mode={mode},synth={kind},seed=77",
                            b"")
        assert struct.unpack("<Q", out.tobytes())[0] == O.digest_u16(r_out)
        assert int(params["lo"]) == r_st["lo"] and int(params["hi"]) == r_st["hi"]
        assert params["synth"] == kind and params["seed"] == "77"
        _, lut = G.run("LUT_GEN", f"rows={rows},cols={cols},mode={mode},synth={kind},seed=77", b"")
        assert lut.tobytes() == r_lut.tobytes()
    finally:
        G.init([0])


@pytest.mark.gpu
@pytest.mark.parametrize("prec,name", [(O.PREC_F32, "f32"), (O.PREC_BF16, "bf16"), (O.PREC_TF32, "tf32")])
@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_synth_matmul_samples(gpu, prec, name, devices):
    m, k, n = 4100, 4097, 4104  # 2^37 flop: sharded over 2 bound devices
    try:
        G.init(devices)
        params, out = G.run("MATMUL", f"m={m},k={k},n={n},prec={name},synth=uniform32,seed=5,samples=300",
                            b"")
    finally:
        G.init([0])
    assert params["samples"] == "300" and out.nbytes == 300 * 12
    _check_samples(_samples(out.tobytes()), O.MAT_UNIFORM32, 5, m, k, n, prec)


@pytest.mark.gpu
@pytest.mark.slow
def test_c3_and_c4_through_the_server(gpu, refl):
    """The over-cap configs through the served path (reference client ->
    B200 server, header-only requests): C3 LUT_CORRECT 32768^2 -> digest ==
    the oracle's; C4 MATMUL 32768^3 bf16 -> 16 samples within 1e-5 of the
    f64 oracle on bf16-rounded operands."""
    with G.Server(max_tasks=2) as s:
        st, params, blob, _ = refl.ref_submit(
            s.port, "LUT_CORRECT", f"rows=32768,cols=32768,synth=ramp12,seed={SEED}", b"")
        assert st == "OK", params
        scene = O.synth_image(O.IMG_RAMP12, SEED, 32768, 32768)
        r_out, _, r_st = O.lut_correct(scene, O.LUT_EQUALIZE)
        del scene
        assert struct.unpack("<Q", blob)[0] == O.digest_u16(r_out)
        del r_out
        assert int(G.parse_params(params)["cdf_min"]) == r_st["cdf_min"]
        st, params, blob, _ = refl.ref_submit(
            s.port, "MATMUL", f"m=32768,k=32768,n=32768,prec=bf16,synth=uniform32,seed={SEED},samples=16",
            b"")
        assert st == "OK", params
    samples = _samples(blob)
    rows = sorted({r for r, _, _ in samples})
    A = {r: O.round_matrix(O.PREC_BF16, O.synth_matrix(O.MAT_UNIFORM32, SEED, 32768, 32768, r, 1))[0]
         .astype(np.float64) for r in rows}
    B = O.round_matrix(O.PREC_BF16, O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(SEED), 32768, 32768))
    for r, c, v in samples:
        b = B[:, c].astype(np.float64)
        assert abs(v - float(A[r] @ b)) <= 1e-5 * float(np.abs(A[r]) @ np.abs(b))
