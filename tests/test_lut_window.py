"""The count pass's u32 window (lut.cu WindowCounter): when the layout
sample's values span < 16384 - 2048, every value in a 16384-value window
centred on them gets its own u32 smem counter (red.shared, no wrap test);
values outside it go to the packed histogram, and fold_window() moves the
window into the packed histogram (low 16 bits) and the overflow counters
(the rest) before the partial flush.  Bit-exact against the oracle for:
outliers outside the window in otherwise narrow data (mixed warps), a
window clamped at the top of the u16 range, window bins past 65535 counts
per CTA (the fold's overflow booking), with and without the residual
plane, and through LUT_GEN (count pass only)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _dev():
    import torch
    from paper_1505_05655_b200 import device as D
    return torch, D


def u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16).ravel()


def _check(vals: np.ndarray, plane: bool):
    torch, D = _dev()
    img = torch.from_numpy(vals.view(np.int16)).cuda()
    n = vals.size
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    lut, stats = D.new_lut(), D.new_stats()
    ws = D.lut_workspace(n) if plane else D.lut_workspace(1)
    out = torch.empty_like(img)
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st
    # LUT_GEN: the count pass alone (+ LUT)
    lut2, stats2 = D.new_lut(), D.new_stats()
    D.lut_gen(img, O.LUT_EQUALIZE, lut2, stats2, ws)
    assert np.array_equal(u16(lut2), ref_lut) and D.read_stats(stats2) == ref_st


def _noisy_ramp(n: int, lo: int, span: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    base = lo + (np.arange(n, dtype=np.int64) * span) // n
    return (base + rng.integers(0, 64, n)).astype(np.uint16)


@pytest.mark.parametrize("plane", [True, False])
def test_window_with_outliers(gpu, plane):
    """Narrow data with sparse outliers far outside any window: warps with
    an outlier take the per-sample route (window or packed histogram)."""
    n = (1 << 25) + 4097
    vals = _noisy_ramp(n, 20000, 3000, 1)
    rng = np.random.default_rng(2)
    idx = rng.integers(0, n, n // 997)
    vals[idx] = rng.choice(np.array([0, 1, 65534, 65535, 5000, 50000], dtype=np.uint16), idx.size)
    _check(vals, plane)


@pytest.mark.parametrize("plane", [True, False])
def test_window_at_top_of_range(gpu, plane):
    """Sampled values near 65535: the window is clamped to [49152, 65536)."""
    n = (1 << 25) + 33
    vals = _noisy_ramp(n, 65535 - 3000 - 64, 3000, 3)
    _check(vals, plane)


@pytest.mark.parametrize("plane", [True, False])
def test_window_counts_past_65535_per_cta(gpu, plane):
    """Three interleaved values (no equal neighbours, so not the repetitive
    path): each window counter reaches ~90k per CTA, the fold books the part
    above 16 bits into the overflow counters."""
    n = 40_000_000
    vals = np.empty(n, dtype=np.uint16)
    vals[0::3] = 1000
    vals[1::3] = 1001
    vals[2::3] = 77
    _check(vals, plane)


def test_window_reuse_and_both_window_edges(gpu):
    """Values exactly at the window's first and last counters, the workspace
    reused for a second image (overflow counters self-cleaning)."""
    torch, D = _dev()
    n = (1 << 25) + 1
    a = _noisy_ramp(n, 30000, 2000, 4)
    # the window is centred on the sampled range [~30000, ~32063]: lo ~ 22844
    a[::5000] = 22000          # below the window (packed path)
    a[1::5000] = 40000         # above it
    b = _noisy_ramp(n, 100, 5000, 5)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    for vals in (a, b):
        img = torch.from_numpy(vals.view(np.int16)).cuda()
        ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
        out = torch.empty_like(img)
        D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
        assert np.array_equal(u16(out), ref_out)
        assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st
