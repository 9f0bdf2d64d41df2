"""LSQ_POLYFIT on the B200 vs the REFERENCE's own f64 normal-equation fit
(proj/src/lsq.cpp, compiled into oracle/_ref), compared as whole response
frames: coefficients and SSE bit-identical, errors (order too high,
non-finite samples, too few points, bad dtype) identical.  Cases follow
the reference's tests (test_lsq.cpp, acceptance.cpp:278-315 / 422-425:
6 scan lines x 6000 pixels, orders 1-3) plus orders up to 8, f32 input,
and multi-chunk lines (> 4096 pixels, exercising the fixed-chunk
reduction order)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1505_05655_b200 as G
import wire_util as W


def _frame(lines, pixels, order, y: np.ndarray, dtype="f64"):
    params = f"lines={lines},pixels={pixels},order={order}" + (f",dtype={dtype}" if dtype != "f64" else "")
    return W.frame("LSQ_POLYFIT", params, y.astype(np.float32 if dtype == "f32" else np.float64).tobytes(),
                   "fits.bin")


@pytest.mark.parametrize("req", [
    W.header("LSQ_POLYFIT", "lines=6,pixels=6000", has_payload=True),          # missing order
    W.header("LSQ_POLYFIT", "lines=6,pixels=6000,order=2,dtype=f16", has_payload=True),
    W.header("LSQ_POLYFIT", "lines=0,pixels=6000,order=2", has_payload=True),
    W.header("LSQ_POLYFIT", "lines=100000,pixels=100000,order=2", has_payload=True),
    W.frame("LSQ_POLYFIT", "lines=1,pixels=16,order=9", np.ones(16).tobytes()),  # OrderTooHigh
    W.frame("LSQ_POLYFIT", "lines=1,pixels=1,order=0", np.ones(1).tobytes()),    # pixels < 2
])
def test_lsq_errors_equal_reference(refl, req):
    assert G.handle_request(req) == refl.ref_handle_request(req)


def _lines(rng, lines, pixels, order, noise=1e-3):
    x = np.arange(pixels, dtype=np.float64)
    out = []
    for _ in range(lines):
        c = rng.normal(size=order + 1) / (float(max(pixels, 2)) ** np.arange(order + 1))
        out.append(np.polyval(c[::-1], x) + noise * rng.normal(size=pixels))
    return np.concatenate(out)


@pytest.mark.gpu
@pytest.mark.parametrize("order", [0, 1, 2, 3, 5, 8])
@pytest.mark.parametrize("lines,pixels", [(6, 6000), (1, 2), (3, 17), (2, 4096), (2, 4097),
                                          (4, 20000)])
def test_fits_bit_identical_to_reference(gpu, refl, order, lines, pixels):
    rng = np.random.default_rng(order * 131 + pixels)
    y = _lines(rng, lines, pixels, order)
    req = _frame(lines, pixels, order, y)
    ours = G.handle_request(req)
    ref = refl.ref_handle_request(req)
    assert W.parse_response(ours)["status"] == W.parse_response(ref)["status"]
    assert ours == ref


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 3])
def test_f32_input_bit_identical(gpu, refl, order):
    y = _lines(np.random.default_rng(9), 6, 6000, order).astype(np.float32)
    req = _frame(6, 6000, order, y, dtype="f32")
    assert G.handle_request(req) == refl.ref_handle_request(req)


@pytest.mark.gpu
def test_non_finite_and_insufficient_lines_report_like_reference(gpu, refl):
    y = _lines(np.random.default_rng(4), 3, 50, 2)
    y[50 + 17] = np.nan  # line 1
    y[2 * 50 + 3] = np.inf
    req = _frame(3, 50, 2, y)
    ours, ref = G.handle_request(req), refl.ref_handle_request(req)
    assert W.parse_response(ours)["status"] == "ERR:TASK_FAILED"
    assert ours == ref
    req = _frame(2, 4, 5, np.ones(8))  # 4 points for order 5
    assert G.handle_request(req) == refl.ref_handle_request(req)


@pytest.mark.gpu
def test_recovers_exact_polynomial(gpu):
    x = np.arange(6000, dtype=np.float64)
    coeffs = np.array([3.0, -2e-3, 5e-7])
    y = np.tile(coeffs[0] + coeffs[1] * x + coeffs[2] * x * x, 6)
    resp = W.parse_response(G.handle_request(_frame(6, 6000, 2, y)))
    fits = np.frombuffer(resp["payload"], dtype=np.float64).reshape(6, 4)
    assert np.allclose(fits[:, :3], coeffs, rtol=1e-6, atol=1e-9)
    assert np.all(fits[:, 3] < 1e-12)
    assert G.parse_params(resp["params"]) == {"lines": "6", "order": "2", "bytes": str(6 * 4 * 8)}
