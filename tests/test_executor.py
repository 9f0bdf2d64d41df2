"""The B200 executor's request handling vs the REFERENCE's, byte for byte.

Both sides serve one request held in memory -- srv::handle_connection over
a wire::MemoryStream (the reference pattern of tests/test_server.cpp:65-188):
  ours : gpcx_handle_request        (libgpcx.so: B200 registry)
  ref  : the reference gpc compiled from its own sources, whose registry holds
         its builtins plus the CPU-restated LUT / MATMUL descriptors
         (oracle/ref_shim.cpp)
Every failure path must produce the identical response frame (status code,
msg text, echoed output name): the reference's error mapping
(proj/src/registry.cpp:38-77), early reject before the payload
(proj/src/server.cpp:73-93) and header salvage (server.cpp:15-24).  With a
GPU, valid LUT requests must produce byte-identical OK frames too.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import paper_1505_05655_b200 as G
import wire_util as W
from conftest import has_gpu

FLAGS = ["LUT_GEN", "LUT_APPLY", "LUT_CORRECT", "MATMUL"]


def both(refl, req: bytes):
    return G.handle_request(req), refl.ref_handle_request(req)


ERROR_CASES = [
    W.header("NO_SUCH_TASK", "rows=4,cols=4"),
    W.header("LUT_CORRECT", "rows=4", has_payload=True),
    W.header("LUT_CORRECT", "rows=abc,cols=4", has_payload=True),
    W.header("LUT_CORRECT", "==,,", has_payload=True),
    W.header("LUT_CORRECT", "rows=32768,cols=32768", has_payload=True),
    W.header("LUT_CORRECT", "rows=0,cols=4", has_payload=True),
    W.header("LUT_CORRECT", "rows=4,cols=4"),                         # no marker
    W.header("LUT_CORRECT", "rows=4,cols=4,dtype=f32", has_payload=True),
    W.header("LUT_CORRECT", "rows=4,cols=4,mode=gamma", has_payload=True),
    W.header("LUT_APPLY", "rows=16384,cols=32768", has_payload=True),
    W.header("MATMUL", "m=4,k=4", has_payload=True),
    W.header("MATMUL", "m=4,k=4,n=4,prec=f16", has_payload=True),
    W.header("MATMUL", "m=16384,k=16384,n=16384", has_payload=True),
    W.header("MATMUL", "m=0,k=0,n=0", has_payload=True),
    W.header("MATMUL", "m=65536,k=1,n=65536", has_payload=True),       # response over cap
    W.header("LUT_GEN", "rows=4,rows=4", has_payload=True),            # duplicate key
    W.header("LUT_GEN", "Rows=4,cols=4", has_payload=True),            # bad key
    W.header("LUT_GEN", "rows=4,cols=4", marker=0x41),                 # bad marker
    W.header("LUT_GEN", "rows=4,cols=4", name="x" * 29 + "\x01"),      # bad name char
    W.header("\x07UT_GEN", "rows=4,cols=4", name="saved.bin"),         # salvage name
    W.header("", "", name=""),
]


@pytest.mark.parametrize("i", range(len(ERROR_CASES)))
def test_error_responses_identical_to_reference(refl, i):
    ours, ref = both(refl, ERROR_CASES[i])
    assert W.parse_response(ours)["status"].startswith("ERR:")
    assert ours == ref, (W.parse_response(ours), W.parse_response(ref))


def test_payload_length_mismatch_identical(refl):
    for flag, params, n in [("LUT_CORRECT", "rows=4,cols=4", 30), ("LUT_APPLY", "rows=2,cols=2", 8),
                            ("MATMUL", "m=2,k=2,n=2", 15)]:
        req = W.header(flag, params, has_payload=True) + bytes(n)
        # the stream holds fewer bytes than promised -> truncated on both
        with pytest.raises(G.GpcxError) as e:
            G.handle_request(req)
        assert e.value.code == "Truncated"
        with pytest.raises(refl.RefError) as r:
            refl.ref_handle_request(req)
        assert r.value.status == 10  # Errc::Truncated + 1


def test_dispatch_fuzz_never_throws_and_matches_reference(refl):
    """The 500-frame fuzz of test_registry.cpp:329-355, run through both
    servers' handle_connection, on the error paths a CPU box can take."""
    rng = random.Random(0xD15EA5E)
    for _ in range(500):
        flag = rng.choice(FLAGS + ["WHAT", ""]) if rng.random() < 0.7 else W.printable(rng, 29)
        params = W.printable(rng, 200)
        if rng.random() < 0.25:
            params = rng.choice(["rows=4,cols=4", "m=2,k=2,n=2", "rows=4,cols=4,mode=stretch"])
        name = W.printable(rng, 30)
        marker = rng.choice([W.MARK_DATA, W.MARK_NONE])
        payload = bytes([0x5A]) * rng.randint(0, 64) if marker == W.MARK_DATA else b""
        req = W.header(flag, params, name, marker=marker) + payload
        try:
            ours = G.handle_request(req)
        except G.GpcxError as e:
            assert e.code == "Truncated"
            with pytest.raises(refl.RefError):
                refl.ref_handle_request(req)
            continue
        r = W.parse_response(ours)
        assert r["status"] == "OK" or r["status"].startswith("ERR:")
        ref = refl.ref_handle_request(req)
        if r["status"] == "ERR:TASK_FAILED" and not has_gpu():
            continue  # a valid request on a GPU-less box: no CPU fallback by design
        if W.parse_response(ref)["status"] == "OK" and r["status"] == "OK" and flag == "MATMUL":
            continue  # fp32 GPU vs f64 CPU: compared within tolerance in test_matmul_gpu
        assert ours == ref, (req[:40], r, W.parse_response(ref))


@pytest.mark.gpu
@pytest.mark.parametrize("flag,mode", [("LUT_CORRECT", "equalize"), ("LUT_CORRECT", "stretch"),
                                       ("LUT_GEN", "equalize"), ("LUT_GEN", "stretch")])
def test_valid_lut_requests_byte_identical(gpu, refl, flag, mode):
    from oracle import oracle as O
    rows, cols = 123, 457
    img = O.synth_image(O.IMG_RAMP12, 3, rows, cols)
    req = W.frame(flag, f"rows={rows},cols={cols},mode={mode}", img.tobytes(), "corr.raw")
    ours, ref = both(refl, req)
    assert W.parse_response(ours)["status"] == "OK"
    assert ours == ref


@pytest.mark.gpu
def test_valid_lut_apply_byte_identical(gpu, refl):
    from oracle import oracle as O
    img = O.synth_image(O.IMG_UNIFORM16, 4, 64, 80)
    lut = (np.arange(65536, dtype=np.uint32) * 40503 >> 16).astype(np.uint16)
    req = W.frame("LUT_APPLY", "rows=64,cols=80", lut.tobytes() + img.tobytes())
    ours, ref = both(refl, req)
    assert ours == ref and W.parse_response(ours)["status"] == "OK"
