"""The residual plane of fused_kernel (lut.cu): at >= 2^25 samples with a
workspace of gpcx_lut_workspace_size(n) bytes, the count pass stores every
256-sample block whose samples span < 256 values as (base, one byte per
sample) and the apply pass reads that copy instead of the image.  Results
must be bit-identical to the oracle and to the plane-less path (a workspace
of the fixed size), for every block kind: narrow, wide, range exactly 255 /
256, flat, at the top of the u16 range, MSB-aligned (swizzled layout), and
for unaligned / in-place buffers, odd lengths and reuse of one workspace."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

PLANE_MIN = 1 << 25


def _dev():
    import torch
    from paper_1505_05655_b200 import device as D
    return torch, D


def u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16).ravel()


def fixed_ws(D, n):
    """A workspace of the fixed size only: no room for the plane."""
    return D.lut_workspace(1)


def mixed_image(n: int, seed: int = 7) -> np.ndarray:
    """Blocks of 256 samples with a per-block kind (block boundaries are
    relative to the buffer start; with an unaligned view they straddle the
    kernel's blocks, which is the point of the offsets below)."""
    rng = np.random.default_rng(seed)
    nb = (n + 255) // 256
    kind = rng.integers(0, 8, nb)
    base = rng.integers(0, 65536 - 256, nb)
    out = np.empty(nb * 256, dtype=np.int64)
    blocks = out.reshape(nb, 256)
    r = rng.integers(0, 256, (nb, 256))
    blocks[:] = base[:, None] + r                                          # 0: narrow (range <= 255)
    w = kind == 1
    blocks[w] = rng.integers(0, 65536, (w.sum(), 256))                     # 1: wide
    e = kind == 2                                                          # 2: range exactly 255
    blocks[e] = base[e, None] + r[e] % 256
    blocks[e, 0] = base[e]
    blocks[e, 1] = base[e] + 255
    e = kind == 3                                                          # 3: range exactly 256
    blocks[e] = base[e, None] + r[e] % 256
    blocks[e, 0] = base[e]
    blocks[e, 1] = base[e] + 256
    f = kind == 4
    blocks[f] = base[f, None]                                              # 4: flat
    t = kind == 5
    blocks[t] = 65535 - r[t] % 256                                         # 5: top of the range
    blocks[t, 0] = 65535
    z = kind == 6
    blocks[z] = r[z] % 200                                                 # 6: near zero
    return out[:n].astype(np.uint16)


@pytest.mark.parametrize("off", [0, 1, 3, 7])
def test_plane_mixed_blocks_bit_exact(gpu, off):
    torch, D = _dev()
    n = PLANE_MIN + 12_345  # not a whole number of blocks
    vals = mixed_image(n + 8)
    dev = torch.from_numpy(vals.view(np.int16)).to(gpu)
    src = dev[off:off + n]
    ref_out, ref_lut, ref_st = O.lut_correct(vals[off:off + n], O.LUT_EQUALIZE)
    lut, stats = D.new_lut(), D.new_stats()
    ws = D.lut_workspace(n)
    assert ws.numel() > fixed_ws(D, n).numel()  # room for the plane
    out = torch.zeros(n + 8, dtype=torch.int16, device=gpu)[off:off + n]  # co-aligned with src
    D.lut_correct(src, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st
    # the plane-less path: same bytes
    out2 = torch.zeros(n + 8, dtype=torch.int16, device=gpu)[off:off + n]
    D.lut_correct(src, out2, O.LUT_EQUALIZE, lut, stats, fixed_ws(D, n))
    assert torch.equal(out, out2)


def test_plane_in_place_and_workspace_reuse(gpu):
    torch, D = _dev()
    n = PLANE_MIN + 999
    lut, stats = D.new_lut(), D.new_stats()
    ws = D.lut_workspace(n)
    for seed in (1, 2):
        vals = mixed_image(n, seed)
        img = torch.from_numpy(vals.view(np.int16)).to(gpu)
        ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
        D.lut_correct(img, img, O.LUT_EQUALIZE, lut, stats, ws)  # in place
        assert np.array_equal(u16(img), ref_out)
        assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
def test_plane_synthetic_scenes(gpu, kind):
    """ramp12 codes every block, uniform16 none: both exact."""
    torch, D = _dev()
    rows, cols = 8192, 4100
    img = D.synth_image(kind, 0x5EED, rows, cols)
    ref_out, ref_lut, ref_st = O.lut_correct(u16(img), O.LUT_EQUALIZE)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


@pytest.mark.parametrize("shift", [4, 8])
def test_plane_msb_aligned(gpu, shift):
    """MSB-aligned data takes the swizzled smem layouts: coded blocks go
    through the swizzled LUT lookups too."""
    torch, D = _dev()
    n = PLANE_MIN + 77
    rng = np.random.default_rng(shift)
    # narrow blocks in units of 2^shift (range < 256 only for shift 4 with small steps)
    steps = (np.arange(n) // 4096) % (4096 >> shift)
    vals = ((steps + rng.integers(0, 4, n)) << shift).astype(np.uint16)
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


def test_plane_flat_and_binary_scenes(gpu):
    """Repetitive data takes the kFew count variant: coded too."""
    torch, D = _dev()
    n = PLANE_MIN + 5
    for vals in (np.full(n, 4242, dtype=np.uint16),
                 np.where((np.arange(n) // 1000) % 2 == 0, 300, 40000).astype(np.uint16)):
        img = torch.from_numpy(vals.view(np.int16)).to(gpu)
        ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
        out = torch.empty_like(img)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
        D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
        assert np.array_equal(u16(out), ref_out)
        assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


@pytest.mark.parametrize("shift", [2, 4, 8])
@pytest.mark.parametrize("outliers", [False, True])
def test_plane_and_window_shifted_for_msb_aligned_smooth_data(gpu, shift, outliers):
    """Smooth MSB-aligned data (a ramp in steps of 2^shift): the layout
    sample picks the shifted u32 window (counter v >> shift) and the shifted
    plane (residual (v - base) >> shift); off-grid samples fall back to the
    packed bins / raw blocks."""
    torch, D = _dev()
    n = PLANE_MIN + 4099
    rng = np.random.default_rng(shift)
    span = 3000 if shift < 8 else 200
    base = (np.arange(n, dtype=np.int64) * span) // n + rng.integers(0, 40, n)
    vals = (np.minimum(base, (65535 >> shift)) << shift).astype(np.uint16)
    if outliers:
        idx = rng.integers(0, n, n // 5000)
        vals[idx] = vals[idx] | 1   # off the 2^shift grid
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_plane_threshold(gpu, delta):
    """Just below / at / above 2^25 samples (the plane starts at 2^25): the
    same bytes as the oracle either way."""
    torch, D = _dev()
    n = PLANE_MIN + delta
    img = D.synth_image(O.IMG_RAMP12, 11, 1, n)
    ref_out, ref_lut, ref_st = O.lut_correct(u16(img), O.LUT_EQUALIZE)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st
