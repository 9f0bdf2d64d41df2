"""The drop-in itself: the REFERENCE server (its own handle_connection,
dispatch, registry and TCP code) with the B200 plugin of
integration/gpc_b200_tasks.cpp registered next to its built-in tasks,
exactly as INTEGRATION.md tells a maintainer to do.  Built from the
reference's sources into oracle/_ref/libgpc_b200_ref.so (test harness).

Checks: the reference registry now lists the GPU flags beside its
builtins; its answers equal the B200 executor's own answers byte-for-byte
(errors on CPU; OK payloads on the GPU); the reference client round-trips
through the reference server onto the GPU."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import paper_1505_05655_b200 as G
import wire_util as W

LIB = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "libgpc_b200_ref.so"


@pytest.fixture(scope="module")
def refb():
    if not LIB.exists():
        pytest.skip("oracle/_ref/libgpc_b200_ref.so not built (needs /root/reference at build time)")
    lib = C.CDLL(str(LIB))
    lib.refb_flags.argtypes = [C.c_char_p, C.c_size_t]
    lib.refb_handle_request.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                        C.POINTER(C.c_size_t)]
    lib.refb_server_start.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_uint16)]
    lib.refb_server_stop.argtypes = [C.c_void_p]
    lib.refb_last_error.restype = C.c_char_p
    return lib


def refb_request(lib, req: bytes) -> bytes:
    cap = max(1 << 16, 4 * len(req) + 4096)
    buf = np.empty(cap, dtype=np.uint8)
    n = C.c_size_t(0)
    src = np.frombuffer(req, dtype=np.uint8)
    rc = lib.refb_handle_request(src.ctypes.data, len(req), buf.ctypes.data, cap, C.byref(n))
    assert rc == 0, lib.refb_last_error()
    return buf[: n.value].tobytes()


def test_reference_registry_gains_gpu_flags(refb):
    buf = C.create_string_buffer(512)
    assert refb.refb_flags(buf, 512) == 0
    flags = buf.value.decode().split(",")
    assert flags == sorted(["BAYER_BILINEAR", "BAYER_GRADIENT", "DEVINFO", "LSQ_POLYFIT",
                            "LUT_APPLY", "LUT_CORRECT", "LUT_GEN", "MATMUL"])


@pytest.mark.parametrize("req", [
    W.header("LUT_CORRECT", "rows=4", has_payload=True),
    W.header("LUT_CORRECT", "rows=32768,cols=32768", has_payload=True),
    W.header("LUT_GEN", "rows=2,cols=2,mode=log", has_payload=True),
    W.header("MATMUL", "m=1,k=1,n=1,prec=fp8", has_payload=True),
    W.header("MATMUL", "m=0,k=1,n=1", has_payload=True),
    W.header("LUT_APPLY", "rows=2,cols=2"),
])
def test_plugin_errors_equal_b200_executor(refb, req):
    assert refb_request(refb, req) == G.handle_request(req)


@pytest.mark.gpu
@pytest.mark.parametrize("flag,params", [("LUT_CORRECT", "rows=300,cols=301"),
                                         ("LUT_CORRECT", "rows=300,cols=301,mode=stretch"),
                                         ("LUT_GEN", "rows=300,cols=301"),
                                         ("MATMUL", "m=64,k=96,n=80,prec=bf16"),
                                         ("MATMUL", "m=64,k=96,n=80")])
def test_plugin_ok_equals_b200_executor(gpu, refb, flag, params):
    from oracle import oracle as O
    if flag == "MATMUL":
        A = O.synth_matrix(O.MAT_UNIFORM32, 1, 64, 96)
        B = O.synth_matrix(O.MAT_UNIFORM32, 2, 96, 80)
        payload = A.tobytes() + B.tobytes()
    else:
        payload = O.synth_image(O.IMG_RAMP12, 5, 300, 301).tobytes()
    req = W.frame(flag, params, payload, "r.bin")
    ours = G.handle_request(req)
    assert W.parse_response(ours)["status"] == "OK"
    assert refb_request(refb, req) == ours


@pytest.mark.gpu
def test_reference_client_through_reference_server_onto_gpu(gpu, refb, refl):
    from oracle import oracle as O
    h, port = C.c_void_p(), C.c_uint16()
    assert refb.refb_server_start(2, C.byref(h), C.byref(port)) == 0
    try:
        img = O.synth_image(O.IMG_UNIFORM16, 9, 512, 512)
        st, params, data, name = refl.ref_submit(port.value, "LUT_CORRECT", "rows=512,cols=512",
                                                 img.tobytes(), "eq.raw")
        assert st == "OK" and name == "eq.raw"
        out, _, stt = O.lut_correct(img, O.LUT_EQUALIZE)
        assert data == out.tobytes()
        assert G.parse_params(params)["cdf_min"] == str(stt["cdf_min"])
        # the builtin CPU tasks are still served next to the GPU ones
        st, _, _, _ = refl.ref_submit(port.value, "DEVINFO", "", b"", "d.xml")
        assert st == "OK"
    finally:
        refb.refb_server_stop(h)


@pytest.mark.gpu
def test_gpu_first_reference_registry_serves_demosaic_on_gpu(gpu, refb, refl):
    """make_b200_registry: BAYER_* / DEVINFO on the B200 inside the reference
    server, byte-identical to the reference's own CPU demosaic."""
    refb.refb2_flags.argtypes = [C.c_char_p, C.c_size_t]
    refb.refb2_handle_request.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                          C.POINTER(C.c_size_t)]
    buf = C.create_string_buffer(512)
    refb.refb2_flags(buf, 512)
    assert "LSQ_POLYFIT" in buf.value.decode() and "BAYER_GRADIENT" in buf.value.decode()
    img = np.random.default_rng(3).integers(0, 65536, 200 * 150, dtype=np.uint32).astype(np.uint16)
    req = W.frame("BAYER_GRADIENT", "rows=200,cols=150,phase=GRBG", img.tobytes(), "p.raw")
    cap = 1 << 20
    out = np.empty(cap, dtype=np.uint8)
    n = C.c_size_t(0)
    src = np.frombuffer(req, dtype=np.uint8)
    assert refb.refb2_handle_request(src.ctypes.data, len(req), out.ctypes.data, cap, C.byref(n)) == 0
    gpu_resp = out[: n.value].tobytes()
    assert W.parse_response(gpu_resp)["status"] == "OK"
    assert gpu_resp == refl.ref_handle_request(req)  # the reference's CPU builtin
