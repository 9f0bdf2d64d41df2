"""LUT_GEN / LUT_APPLY / LUT_CORRECT on the B200 vs the CPU oracle:
bit-exact, through the C ABI (device-level and task-level entry points)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1505_05655_b200 as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

MODES = [(O.LUT_EQUALIZE, "equalize"), (O.LUT_STRETCH, "stretch")]


def _dev():
    import torch
    from paper_1505_05655_b200 import device as D
    return torch, D


def u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16).ravel()


@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 5), (37, 53), (512, 512), (1000, 777)])
def test_synth_image_bit_identical(gpu, kind, rows, cols):
    torch, D = _dev()
    d = D.synth_image(kind, 0x5EED, rows, cols)
    assert np.array_equal(u16(d), O.synth_image(kind, 0x5EED, rows, cols))
    band = D.synth_image(kind, 0x5EED, rows, cols, row0=rows // 2, nrows=rows - rows // 2)
    assert np.array_equal(u16(band), O.synth_image(kind, 0x5EED, rows, cols, row0=rows // 2))


@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 4097, 65536 * 3 + 5, 4096 * 4096])
def test_histogram_exact(gpu, kind, n):
    torch, D = _dev()
    img = D.synth_image(kind, 3, 1, n)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    ws = D.lut_workspace(n)
    D.lut_hist(img, hist, ws)
    ref = O.lut_hist(u16(img))
    assert np.array_equal(hist.cpu().numpy().view(np.uint32).astype(np.uint64), ref)
    D.lut_hist(img, hist, ws)  # workspace is self-cleaning: same answer again
    assert np.array_equal(hist.cpu().numpy().view(np.uint32).astype(np.uint64), ref)


def test_histogram_packed_counter_wraps(gpu):
    """Adjacent bins far past 65535 counts per CTA exercise the packed-u16
    overflow booking (low-half carry, high-half wrap, both at once)."""
    torch, D = _dev()
    n = 3_000_000
    vals = np.empty(n, dtype=np.uint16)
    vals[0::3] = 1000   # even bin (low half)
    vals[1::3] = 1001   # odd bin (high half) of the same word
    vals[2::3] = 77
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    ws = D.lut_workspace(n)
    for _ in range(2):
        D.lut_hist(img, hist, ws)
        h = hist.cpu().numpy().view(np.uint32)
        assert h[1000] == h[1001] == h[77] == n // 3
        assert h.sum(dtype=np.uint64) == n
    const = torch.full((5_000_000,), 4242, dtype=torch.int16, device=gpu)
    D.lut_hist(const, hist, D.lut_workspace(const.numel()))
    h = hist.cpu().numpy().view(np.uint32)
    assert h[4242] == 5_000_000 and h.sum(dtype=np.uint64) == 5_000_000


@pytest.mark.parametrize("mode,mname", MODES)
@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
@pytest.mark.parametrize("rows,cols", [(1, 1), (2, 3), (64, 64), (333, 517), (4096, 4096)])
def test_lut_correct_device_bit_exact(gpu, mode, mname, kind, rows, cols):
    torch, D = _dev()
    img = D.synth_image(kind, 0x5EED, rows, cols)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
    D.lut_correct(img, out, mode, lut, stats, ws)
    ref_out, ref_lut, ref_st = O.lut_correct(u16(img), mode)
    assert np.array_equal(u16(lut), ref_lut)
    assert np.array_equal(u16(out), ref_out)
    assert D.read_stats(stats) == ref_st


@pytest.mark.parametrize("mode", [O.LUT_EQUALIZE, O.LUT_STRETCH])
def test_from_hist_and_minmax_paths_agree(gpu, mode):
    torch, D = _dev()
    img = D.synth_image(O.IMG_RAMP12, 1, 300, 300)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    ws = D.lut_workspace(img.numel())
    D.lut_hist(img, hist, ws)
    lut_a, st_a = D.new_lut(), D.new_stats()
    D.lut_from_hist(hist, mode, lut_a, st_a, ws)
    lut_b, st_b = D.new_lut(), D.new_stats()
    D.lut_gen(img, mode, lut_b, st_b, ws)
    assert np.array_equal(u16(lut_a), u16(lut_b))
    ref_lut, _ = O.lut_gen(u16(img), mode)
    assert np.array_equal(u16(lut_a), ref_lut)


@pytest.mark.parametrize("in_off,out_off", [(0, 0), (1, 1), (3, 3), (1, 0), (0, 5)])
def test_apply_unaligned_and_inplace(gpu, in_off, out_off):
    torch, D = _dev()
    n = 100_003
    base = D.synth_image(O.IMG_UNIFORM16, 8, 1, n + 16)
    lut_np = (np.arange(65536, dtype=np.uint32) * 2654435761 >> 16).astype(np.uint16)
    lut = torch.from_numpy(lut_np.view(np.int16)).to(gpu)
    src = base[in_off:in_off + n]
    dst_buf = torch.zeros(n + 16, dtype=torch.int16, device=gpu)
    dst = dst_buf[out_off:out_off + n]
    D.lut_apply(lut, src, dst)
    assert np.array_equal(u16(dst), lut_np[u16(src)])
    inplace = src.clone()
    D.lut_apply(lut, inplace, inplace)
    assert np.array_equal(u16(inplace), lut_np[u16(src)])


@pytest.mark.parametrize("mode", [O.LUT_EQUALIZE, O.LUT_STRETCH])
@pytest.mark.parametrize("in_off,out_off", [(0, 0), (1, 1), (3, 3), (1, 0), (0, 5), (None, None)])
def test_lut_correct_fused_alignment_and_inplace(gpu, in_off, out_off, mode):
    """LUT_CORRECT (equalize: fused_kernel, stretch: stretch_fused_kernel) is
    one cooperative launch when in/out are co-aligned (incl. in place), the
    gen + apply launches otherwise: same bytes."""
    torch, D = _dev()
    n = 1_000_003
    base = D.synth_image(O.IMG_RAMP12, 9, 1, n + 16)
    if in_off is None:  # in place
        src = base[3:3 + n].clone()
        ref_out, ref_lut, ref_st = O.lut_correct(u16(src), mode)
        dst = src
    else:
        src = base[in_off:in_off + n]
        ref_out, ref_lut, ref_st = O.lut_correct(u16(src), mode)
        dst = torch.zeros(n + 16, dtype=torch.int16, device=gpu)[out_off:out_off + n]
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    D.lut_correct(src, dst, mode, lut, stats, ws)
    assert np.array_equal(u16(dst), ref_out)
    assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st


@pytest.mark.parametrize("mode,mname", MODES)
def test_sharded_correct_from_summed_band_histograms(gpu, mode, mname):
    """The N-GPU step on one device: per-band histograms (count stage),
    summed like the all-reduce, then LUT + apply per band
    (gpcx_lut_correct_from_hist_device) == the whole-image oracle."""
    torch, D = _dev()
    rows, cols = 1001, 777
    img = D.synth_image(O.IMG_RAMP12, 12, rows, cols)
    ref_out, ref_lut, ref_st = O.lut_correct(u16(img), mode)
    per = (rows + 2) // 3
    bands = [img[r * cols:min(rows, r + per) * cols] for r in range(0, rows, per)]
    total = torch.zeros(65536, dtype=torch.int64, device=gpu)
    ws = D.lut_workspace(img.numel())
    for b in bands:
        h = torch.zeros(65536, dtype=torch.int32, device=gpu)
        D.lut_hist(b, h, ws)
        total += h.to(torch.int64)
    hist = total.to(torch.int32)
    out = torch.empty_like(img)
    outs = [out[r * cols:min(rows, r + per) * cols] for r in range(0, rows, per)]
    for b, o in zip(bands, outs):
        lut, stats = D.new_lut(), D.new_stats()
        D.lut_correct_from_hist(hist, mode, b, o, lut, stats, ws)
        assert np.array_equal(u16(lut), ref_lut) and D.read_stats(stats) == ref_st
    assert np.array_equal(u16(out), ref_out)


def test_lut_correct_fused_counter_wraps_and_reuse(gpu):
    """Packed-counter wraps through the fused path, twice on one workspace
    (the overflow counters must come back zeroed)."""
    torch, D = _dev()
    n = 3_000_000
    vals = np.empty(n, dtype=np.uint16)
    vals[0::3] = 1000
    vals[1::3] = 1001
    vals[2::3] = 77
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    for _ in range(2):
        out = torch.empty_like(img)
        D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
        assert np.array_equal(u16(out), ref_out) and np.array_equal(u16(lut), ref_lut)
        assert D.read_stats(stats) == ref_st


def test_constant_and_two_level_images(gpu):
    torch, D = _dev()
    for vals in ([1234] * 1000, [300] * 700 + [40000] * 333, [0] * 10 + [65535] * 10):
        arr = np.array(vals, dtype=np.uint16)
        img = torch.from_numpy(arr.view(np.int16)).to(gpu)
        for mode, _ in MODES:
            out = torch.empty_like(img)
            lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
            D.lut_correct(img, out, mode, lut, stats, ws)
            r_out, r_lut, r_st = O.lut_correct(arr, mode)
            assert np.array_equal(u16(out), r_out) and np.array_equal(u16(lut), r_lut)
            assert D.read_stats(stats) == r_st


def test_digest_matches_oracle(gpu):
    torch, D = _dev()
    img = D.synth_image(O.IMG_UNIFORM16, 5, 777, 1001)
    d = D.digest_u16(img, 12345)
    assert int(d.item()) & (2 ** 64 - 1) == O.digest_u16(u16(img), 12345)
    for off in (1, 3, 7, 8):  # unaligned starts: scalar head, 128-bit body, tail
        d = D.digest_u16(img[off:], off)
        assert int(d.item()) & (2 ** 64 - 1) == O.digest_u16(u16(img)[off:], off), off


@pytest.mark.slow
@pytest.mark.parametrize("mode,mname", MODES)
@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
def test_c3_full_size_via_digest(gpu, mode, mname, kind):
    """32768^2 (config C3) LUT_CORRECT on one device, both modes, on the
    bench scene (ramp12) and on uniform16 noise (the worst case for smem
    bank conflicts): checked against the oracle through the position-keyed
    digest (size-independent property) plus the exact LUT and stats."""
    torch, D = _dev()
    rows = cols = 32768
    img = D.synth_image(kind, 0x5EED, rows, cols)
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
    D.lut_correct(img, out, mode, lut, stats, ws)
    host_img = u16(img)
    del img
    r_out, r_lut, r_st = O.lut_correct(host_img, mode)
    del host_img
    assert np.array_equal(u16(lut), r_lut)
    assert D.read_stats(stats) == r_st
    assert int(D.digest_u16(out).item()) & (2 ** 64 - 1) == O.digest_u16(r_out)


@pytest.mark.slow
@pytest.mark.parametrize("mode,mname", MODES)
@pytest.mark.parametrize("pattern", ["flat", "binary", "sparse"])
def test_c3_full_size_degenerate_images(gpu, mode, mname, pattern):
    """The C3 size (2^30 pixels) on the images that stress the count pass's
    special paths hardest: one value everywhere (every CTA's bin wraps its
    u16 half-word ~110 times; the warp-combining path), two values (the
    binary path) and 8 values spread over the range.  Expected LUT / stats
    from the oracle on the exact u64 histogram; out == LUT[in] everywhere."""
    torch, D = _dev()
    rows = cols = 32768
    n = rows * cols
    hist = np.zeros(65536, dtype=np.uint64)
    if pattern == "flat":
        img = torch.full((n,), 12345, dtype=torch.int16, device="cuda")
        hist[12345] = n
    elif pattern == "binary":
        img = torch.full((n,), 1000, dtype=torch.int16, device="cuda")
        img[n // 3:] = 30000
        hist[1000], hist[30000] = n // 3, n - n // 3
    else:
        vals = torch.tensor([7, 4095, 4096, 20000, 32767, 100, 2, 31000], dtype=torch.int16, device="cuda")
        img = vals.repeat(n // 8)
        for v in vals.tolist():
            hist[v] = n // 8
    out = torch.empty_like(img)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    D.lut_correct(img, out, mode, lut, stats, ws)
    r_lut, r_st = O.lut_from_hist(hist, mode)
    assert np.array_equal(u16(lut), r_lut)
    assert D.read_stats(stats) == r_st
    lut_t = torch.from_numpy(r_lut.astype(np.int32)).cuda()
    for a, b in zip(img.split(1 << 28), out.split(1 << 28)):
        want = lut_t[a.to(torch.int32) & 0xFFFF].to(torch.int16)
        assert torch.equal(b, want)


# ----------------------------------------------------------- task level ---

@pytest.mark.parametrize("mode,mname", MODES)
def test_gpcx_run_lut_tasks(gpu, mode, mname):
    rows, cols = 257, 1031
    img = O.synth_image(O.IMG_RAMP12, 42, rows, cols)
    params = f"rows={rows},cols={cols},mode={mname}"
    res, payload = G.run("LUT_CORRECT", params, img)
    r_out, r_lut, r_st = O.lut_correct(img, mode)
    assert np.array_equal(payload.view(np.uint16), r_out)
    want = {"rows": str(rows), "cols": str(cols), "mode": mname, "lo": str(r_st["lo"]),
            "hi": str(r_st["hi"])}
    if mname == "equalize":
        want["cdf_min"] = str(r_st["cdf_min"])
    assert res == want
    res, payload = G.run("LUT_GEN", params, img)
    assert np.array_equal(payload.view(np.uint16), r_lut) and res == want
    res, payload = G.run("LUT_APPLY", f"rows={rows},cols={cols}",
                         np.concatenate([r_lut, img]))
    assert np.array_equal(payload.view(np.uint16), r_out)
    assert res == {"rows": str(rows), "cols": str(cols)}


def test_gpcx_run_pinned_and_pageable_agree(gpu):
    import ctypes as C
    rows, cols = 2048, 3000  # > staging chunk: exercises the chunk pipeline
    img = O.synth_image(O.IMG_UNIFORM16, 1, rows, cols)
    _, a = G.run("LUT_CORRECT", f"rows={rows},cols={cols}", img)
    p = G.lib.gpcx_pinned_alloc(img.nbytes)
    q = G.lib.gpcx_pinned_alloc(img.nbytes)
    try:
        pin_in = np.ctypeslib.as_array((C.c_uint16 * img.size).from_address(p))
        pin_out = np.ctypeslib.as_array((C.c_uint8 * img.nbytes).from_address(q))
        pin_in[:] = img
        _, b = G.run("LUT_CORRECT", f"rows={rows},cols={cols}", pin_in, out=pin_out)
        assert np.array_equal(a, b)
    finally:
        G.lib.gpcx_pinned_free(p)
        G.lib.gpcx_pinned_free(q)
    r_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
    assert np.array_equal(a.view(np.uint16), r_out)


@pytest.mark.parametrize("mode,mname", MODES)
def test_planner_row_bands_bit_identical(gpu, mode, mname):
    """Bind device 0 several times: the planner then splits the request into
    row bands (one per binding) with the histogram / min-max exchange -- the
    multi-GPU code path -- on one physical GPU.  Output must not depend on
    the band count (parexec invariance contract)."""
    rows, cols = 4099, 4101  # > kShardMinPixels, ragged bands
    img = O.synth_image(O.IMG_UNIFORM16, 77, rows, cols)
    r_out, r_lut, r_st = O.lut_correct(img, mode)
    try:
        for g in (2, 3, 8):
            G.init([0] * g)
            assert G.device_count() == g
            for flag in ("LUT_CORRECT", "LUT_GEN"):
                res, payload = G.run(flag, f"rows={rows},cols={cols},mode={mname}", img)
                want = r_out if flag == "LUT_CORRECT" else r_lut
                assert np.array_equal(payload.view(np.uint16), want), (g, flag)
                assert int(res["lo"]) == r_st["lo"] and int(res["hi"]) == r_st["hi"]
            res, payload = G.run("LUT_APPLY", f"rows={rows},cols={cols}", np.concatenate([r_lut, img]))
            assert np.array_equal(payload.view(np.uint16), r_out)
    finally:
        G.init([0])


def test_task_errors_map_to_errc(gpu):
    with pytest.raises(G.GpcxError) as e:
        G.run("LUT_CORRECT", "rows=4,cols=4", np.zeros(15, dtype=np.uint16))
    assert e.value.code == "PayloadMismatch"
    with pytest.raises(G.GpcxError) as e:
        G.run("LUT_CORRECT", "rows=4,cols=4,mode=log", np.zeros(16, dtype=np.uint16))
    assert e.value.code == "BadValue"


@pytest.mark.parametrize("shift", [4, 6, 8])
@pytest.mark.parametrize("rows,cols", [(333, 517), (2048, 4096)])
def test_msb_aligned_images_bit_exact(gpu, shift, rows, cols):
    """MSB-aligned sensor data (12 / 10 / 8 significant bits shifted up):
    every value has trailing zero bits, so the kernels use the swizzled smem
    layout for the histogram and the staged LUT -- histogram, fused
    LUT_CORRECT and the standalone LUT_APPLY kernel must stay bit-exact."""
    torch, D = _dev()
    rng = np.random.default_rng(shift * 1000 + rows)
    vals = ((rng.integers(0, 1 << 16, rows * cols, dtype=np.uint32) >> shift) << shift).astype(np.uint16)
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    ws = D.lut_workspace(img.numel())
    D.lut_hist(img, hist, ws)
    assert np.array_equal(hist.cpu().numpy().view(np.uint32).astype(np.uint64), O.lut_hist(vals))
    for mode, _ in MODES:
        out = torch.empty_like(img)
        lut, stats = D.new_lut(), D.new_stats()
        D.lut_correct(img, out, mode, lut, stats, ws)
        r_out, r_lut, r_st = O.lut_correct(vals, mode)
        assert np.array_equal(u16(out), r_out) and np.array_equal(u16(lut), r_lut), mode
        assert D.read_stats(stats) == r_st
        out2 = torch.empty_like(img)
        D.lut_apply(lut, img, out2)
        assert np.array_equal(u16(out2), r_out)


def test_swizzled_and_flat_counter_wraps(gpu):
    """Counts far past 65535 per CTA in the swizzled layout (few MSB-aligned
    values, combined per warp) and in flat runs (one atomic per warp vector,
    k = 8 x active lanes), including runs that end mid-vector and mid-warp."""
    torch, D = _dev()
    n = 4_000_003
    vals = np.empty(n, dtype=np.uint16)
    vals[0::3] = 0x1000
    vals[1::3] = 0x2000
    vals[2::3] = 0xF000
    vals[: n // 2] = np.where(np.arange(n // 2) % 97 < 90, 0x4000, vals[: n // 2])  # flat runs
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    for _ in range(2):  # the overflow counters must come back zeroed
        D.lut_hist(img, hist, ws)
        assert np.array_equal(hist.cpu().numpy().view(np.uint32).astype(np.uint64), O.lut_hist(vals))
        out = torch.empty_like(img)
        D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
        assert np.array_equal(u16(out), ref_out) and np.array_equal(u16(lut), ref_lut)
        assert D.read_stats(stats) == ref_st


@pytest.mark.parametrize("variant", ["plain", "plain_swizzled", "few", "few_swizzled", "few_random",
                                     "few_random_swizzled", "plain_wide", "few_wide",
                                     "few_random_wide"])
def test_counter_wraps_every_count_variant(gpu, variant):
    """Each count-pass variant (smem layout plain / swizzled x repetitive-
    data probe off / on x the u32 window for narrow data, picked per launch
    from a fixed sample) with > 65535 samples of a value per CTA, so the
    packed u16 halves wrap (or, in the window, the fold books counts above
    16 bits into the overflow counters).  [1000, 1001]: narrow -> the
    window; [1000, 40001]: too wide for it -> the packed plain / few paths."""
    torch, D = _dev()
    n = 24_000_007  # 2 values over 148 CTAs: ~81K samples of each per CTA
    # swizzle strength from the trailing zeros: 0x3008 -> 3 (layout 1),
    # 0x3100 -> 8 (layout 2)
    base = np.array([0x3000, 0x3100] if variant == "few_random_swizzled" else
                    [0x3000, 0x3008] if "swizzled" in variant else
                    [1000, 40001] if "wide" in variant else [1000, 1001], dtype=np.uint16)
    if variant.startswith("plain"):
        vals = base[np.arange(n) % 2]               # adjacent samples always differ
    elif "random" in variant:                        # binary noise: the min/max path
        vals = base[np.random.default_rng(5).integers(0, 2, n)]
    else:
        vals = base[(np.arange(n) // 37) % 2]       # runs of 37: flat + binary vectors
    img = torch.from_numpy(vals.view(np.int16)).to(gpu)
    hist = torch.zeros(65536, dtype=torch.int32, device=gpu)
    ws = D.lut_workspace(n)
    ref_h = O.lut_hist(vals)
    assert ref_h.min(where=ref_h > 0, initial=n) > 148 * 65536  # > 65535 per value per CTA
    D.lut_hist(img, hist, ws)
    assert np.array_equal(hist.cpu().numpy().view(np.uint32).astype(np.uint64), ref_h)
    ref_out, ref_lut, ref_st = O.lut_correct(vals, O.LUT_EQUALIZE)
    out = torch.empty_like(img)
    lut, stats = D.new_lut(), D.new_stats()
    D.lut_correct(img, out, O.LUT_EQUALIZE, lut, stats, ws)
    assert np.array_equal(u16(out), ref_out) and np.array_equal(u16(lut), ref_lut)
    assert D.read_stats(stats) == ref_st


@pytest.mark.parametrize("kind", [O.IMG_RAMP12, O.IMG_UNIFORM16])
def test_planner_bands_past_the_plane_threshold(gpu, kind):
    """In-process planner with bands >= 2^25 samples: each band's count
    launch codes its residual plane and the band's apply launch (after the
    peer histogram sum) reads it -- same bytes as one device."""
    rows, cols = 8192, 8200  # 2 bands of 4096 x 8200 = 33.6 M samples
    img = O.synth_image(kind, 5, rows, cols)
    r_out, r_lut, r_st = O.lut_correct(img, O.LUT_EQUALIZE)
    try:
        for g in (1, 2):
            G.init([0] * g)
            res, payload = G.run("LUT_CORRECT", f"rows={rows},cols={cols},mode=equalize", img)
            assert np.array_equal(payload.view(np.uint16), r_out), g
            assert int(res["lo"]) == r_st["lo"] and int(res["hi"]) == r_st["hi"]
            res, payload = G.run("LUT_GEN", f"rows={rows},cols={cols},mode=equalize", img)
            assert np.array_equal(payload.view(np.uint16), r_lut), g
    finally:
        G.init([0])
