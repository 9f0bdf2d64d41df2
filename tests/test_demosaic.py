"""BAYER_BILINEAR / BAYER_GRADIENT on the B200 vs the REFERENCE's own
demosaic kernels and its independent gpcref oracles (compiled from
proj/src/demosaic.cpp and proj/reference/reference.cpp into oracle/_ref),
byte-exact -- the parity the reference itself pins in
acceptance.cpp:229-273 (4 phases x random mosaics) and
test_demosaic.cpp:130-307 (hand pixels, rounding, edge clamp, gradient
direction).  Plus DEVINFO: the B200 inventory rendered in the reference's
canonical XML."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_1505_05655_b200 as G
import wire_util as W

PHASES = ["RGGB", "BGGR", "GRBG", "GBRG"]


def _mosaic(rng, rows, cols, bits=16):
    return rng.integers(0, 1 << bits, size=rows * cols, dtype=np.uint32).astype(np.uint16)


# ------------------------------------------------------------ CPU tests ---

def test_payload_rule_matches_reference_builtin(refl):
    for params in ["rows=2048,cols=2048", "rows=0,cols=4", "rows=60000,cols=60000", "rows=4",
                   "rows=4,cols=4,phase=XXXX", "rows=4,cols=4,dtype=f32"]:
        for flag in ("BAYER_BILINEAR", "BAYER_GRADIENT"):
            n = C.c_uint64(0)
            rs = refl.ref.ref_expected_payload_len(flag.encode(), params.encode(), C.byref(n))
            try:
                assert G.payload_len(flag, params) == n.value and rs == 0, params
            except G.GpcxError as e:
                if "cols" not in params:  # MissingParam is raised by dispatch, not the rule
                    assert rs == e.status, (params, rs, e.code)


@pytest.mark.parametrize("req", [
    W.header("BAYER_BILINEAR", "rows=60000,cols=60000", has_payload=True),
    W.header("BAYER_GRADIENT", "rows=4", has_payload=True),
    W.header("BAYER_GRADIENT", "rows=4,cols=4"),
    W.frame("BAYER_BILINEAR", "rows=4,cols=4,dtype=f32", bytes(32)),   # handler rejects dtype
    W.frame("BAYER_BILINEAR", "rows=4,cols=4,phase=XGGB", bytes(32)),  # handler rejects phase
    W.header("DEVINFO", "", has_payload=True) + bytes(4),
])
def test_bayer_and_devinfo_errors_equal_reference(refl, req):
    assert G.handle_request(req) == refl.ref_handle_request(req)


def test_devinfo_xml_format_equals_reference(refl):
    d = G.DeviceInfo()
    d.name = b"NVIDIA B200 <&> test"
    d.compute_capability = b"10.0"
    d.warp_size = 32
    d.total_constant_memory = 65536
    d.total_global_memory = 191_000_000_000
    d.shared_memory_per_block = 49152
    d.clock_rate_khz = 1965000
    d.multi_processor_count = 148
    d.registers_per_block = 65536
    d.max_threads_per_block = 1024
    d.max_grid_size[:] = [2147483647, 65535, 65535]
    d.max_threads_dim[:] = [1024, 1024, 64]
    for devs in ([], [d], [d, d]):
        ours = G.devinfo_render(devs)
        arr = (G.DeviceInfo * max(1, len(devs)))(*devs)
        buf = C.create_string_buffer(1 << 16)
        n = C.c_size_t(0)
        refl.ref.ref_devinfo_render.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t,
                                                C.POINTER(C.c_size_t)]
        assert refl.ref.ref_devinfo_render(arr, len(devs), buf, 1 << 16, C.byref(n)) == 0
        assert ours == buf.value.decode()
    assert "&lt;&amp;&gt;" in G.devinfo_render([d])


# ------------------------------------------------------------ GPU tests ---

def _gpu_demosaic(gradient, phase, img, rows, cols):
    import torch
    from paper_1505_05655_b200 import device as D
    t = torch.from_numpy(img.view(np.int16)).cuda()
    out = D.demosaic(gradient, G.PHASES[phase], t, rows, cols)
    return out.cpu().numpy().view(np.uint16)


@pytest.mark.gpu
@pytest.mark.parametrize("gradient", [False, True])
@pytest.mark.parametrize("phase", PHASES)
def test_random_mosaics_equal_reference_kernel_and_gpcref(gpu, refl, gradient, phase):
    """acceptance.cpp:229-240 pattern: random 64x64 mosaics, all phases."""
    rng = np.random.default_rng(0x100B7AC6 + PHASES.index(phase) + 7 * gradient)
    for _ in range(10):
        img = _mosaic(rng, 64, 64)
        ours = _gpu_demosaic(gradient, phase, img, 64, 64)
        assert np.array_equal(ours, refl.ref_demosaic(gradient, img, 64, 64, phase))
        assert np.array_equal(ours, refl.ref_demosaic(gradient, img, 64, 64, phase, gpcref=True))


@pytest.mark.gpu
@pytest.mark.parametrize("gradient", [False, True])
@pytest.mark.parametrize("rows,cols", [(2, 2), (2, 3), (3, 2), (5, 7), (17, 300), (300, 17),
                                       (257, 513), (1024, 1000), (2048, 2048)])
def test_ragged_sizes_equal_reference(gpu, refl, gradient, rows, cols):
    rng = np.random.default_rng(rows * 1000 + cols)
    for phase in PHASES:
        img = _mosaic(rng, rows, cols, bits=12 if rows % 2 else 16)
        ours = _gpu_demosaic(gradient, phase, img, rows, cols)
        assert np.array_equal(ours, refl.ref_demosaic(gradient, img, rows, cols, phase)), (phase,)


@pytest.mark.gpu
def test_hand_computed_pixels_and_edge_clamp(gpu):
    """test_demosaic.cpp:130-205 style: a 4x4 RGGB mosaic with distinct
    values; interior and corner pixels computed by hand."""
    img = np.arange(1, 17, dtype=np.uint16) * 100  # row-major 4x4
    out = _gpu_demosaic(False, "RGGB", img, 4, 4).reshape(3, 4, 4)
    R, Gp, B = out
    v = img.reshape(4, 4).astype(np.uint32)
    # (1,1) is a B site: R = avg4 of diagonals, G = avg4 of the cross
    assert R[1, 1] == (v[0, 0] + v[0, 2] + v[2, 0] + v[2, 2] + 2) // 4
    assert Gp[1, 1] == (v[0, 1] + v[2, 1] + v[1, 0] + v[1, 2] + 2) // 4
    assert B[1, 1] == v[1, 1]
    # (0,0) is an R site at the corner: N clamps to row 0, W clamps to col 0
    n, s, w, e = v[0, 0], v[1, 0], v[0, 0], v[0, 1]
    assert Gp[0, 0] == (n + s + w + e + 2) // 4
    assert B[0, 0] == (v[0, 0] + v[0, 1] + v[1, 0] + v[1, 1] + 2) // 4
    # (0,1): G in a red row: R from E/W, B from N/S (N clamps)
    assert R[0, 1] == (v[0, 0] + v[0, 2] + 1) // 2
    assert B[0, 1] == (v[0, 1] + v[1, 1] + 1) // 2


@pytest.mark.gpu
def test_gradient_picks_smaller_difference(gpu, refl):
    """test_demosaic.cpp:207-248: a vertical edge makes the horizontal
    gradient large, so G at R/B sites averages N/S."""
    rows, cols = 8, 8
    img = np.zeros((rows, cols), dtype=np.uint16)
    img[:, 4:] = 60000
    img[:, 3] = 30000
    ours = _gpu_demosaic(True, "RGGB", img.ravel(), rows, cols)
    assert np.array_equal(ours, refl.ref_demosaic(True, img.ravel(), rows, cols, "RGGB"))


@pytest.mark.gpu
@pytest.mark.parametrize("flag", ["BAYER_BILINEAR", "BAYER_GRADIENT"])
@pytest.mark.parametrize("phase", ["RGGB", "GBRG"])
def test_served_demosaic_byte_identical_to_reference(gpu, refl, flag, phase):
    rng = np.random.default_rng(5)
    img = _mosaic(rng, 96, 130)
    req = W.frame(flag, f"rows=96,cols=130,phase={phase}", img.tobytes(), "planes.raw")
    ours = G.handle_request(req)
    assert W.parse_response(ours)["status"] == "OK"
    assert ours == refl.ref_handle_request(req)


@pytest.mark.gpu
def test_undersized_image_fails_like_reference(gpu, refl):
    req = W.frame("BAYER_BILINEAR", "rows=1,cols=8", bytes(16))
    assert G.handle_request(req) == refl.ref_handle_request(req)
    assert W.parse_response(G.handle_request(req))["status"] == "ERR:TASK_FAILED"


@pytest.mark.gpu
def test_devinfo_reports_the_b200(gpu):
    devs = G.devinfo_probe()
    assert len(devs) >= 1
    assert b"B200" in devs[0].name and devs[0].compute_capability == b"10.0"
    assert devs[0].multi_processor_count == 148 and devs[0].warp_size == 32
    resp = W.parse_response(G.handle_request(W.header("DEVINFO", "", name="gpu.xml")))
    assert resp["status"] == "OK" and resp["name"] == "gpu.xml"
    xml = resp["payload"].decode()
    assert xml.startswith('<?xml version="1.0"?>\n<gpgpu_server>\n  <device index="0">\n')
    assert "<multi_processor_count>148</multi_processor_count>" in xml
    assert G.parse_params(resp["params"])["devices"] == str(len(devs))


_RPT_CHECK = r"""
import sys, numpy as np
sys.path.insert(0, "tests")
import test_demosaic as T
from oracle import oracle as O
bad = []
for gradient in (False, True):
    for rows, cols in [(31, 264), (32, 256), (33, 257), (63, 520), (64, 512), (65, 130),
                       (127, 776), (129, 2056), (200, 8)]:
        rng = np.random.default_rng(rows * 7 + cols)
        for phase in T.PHASES:
            img = T._mosaic(rng, rows, cols)
            if not np.array_equal(T._gpu_demosaic(gradient, phase, img, rows, cols),
                                  O.ref_demosaic(gradient, img, rows, cols, phase)):
                bad.append((gradient, rows, cols, phase))
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("rpt", ["4", "8"])
def test_both_tile_heights_equal_reference(gpu, refl, rpt):
    """The launcher picks 4 rows per thread (32-row tiles) for bilinear and 8
    (64-row tiles) for gradient; GPCX_DEMOSAIC_RPT forces one height for
    both.  Each height, both kernels, all phases, tile-edge sizes."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, GPCX_DEMOSAIC_RPT=rpt)
    r = subprocess.run([sys.executable, "-c", _RPT_CHECK], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("bands,rows,cols,phase", [
    (2, 4096, 4096, "RGGB"),
    (3, 4099, 4104, "GBRG"),   # uneven bands, odd band starts
    (2, 4100, 4097, "BGGR"),   # odd row length: the scalar store path
])
def test_row_band_sharded_demosaic_equals_reference(gpu, refl, bands, rows, cols, phase):
    """The planner splits large mosaics into row bands (1-row halo each side,
    image-coordinate clamp and CFA parity); the served result must equal the
    reference's whole-image kernel byte for byte."""
    rng = np.random.default_rng(rows ^ cols)
    img = _mosaic(rng, rows, cols)
    try:
        G.init([0] * bands)
        for flag, grad in (("BAYER_BILINEAR", False), ("BAYER_GRADIENT", True)):
            _, out = G.run(flag, f"rows={rows},cols={cols},phase={phase}", img)
            ref = refl.ref_demosaic(grad, img, rows, cols, phase, workers=0)
            assert np.array_equal(out.view(np.uint16), ref), (flag, bands)
    finally:
        G.init([0])
