"""ctypes access to the CPU oracle and to the compiled reference.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product.

  orc  : oracle/_build/liboracle.so  (gpcx_oracle.c, the CPU restatement;
         parity status in gpcx_oracle.h: unpinned by the reference, pinned by
         KATs + tests/oracle_np.py)
  ref  : oracle/_ref/libgpc_ref.so   (the reference gpc compiled from its own
         sources + ref_shim.cpp); None when it was not built
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_PATH = HERE / "_build" / "liboracle.so"
REF_PATH = HERE / "_ref" / "libgpc_ref.so"

LUT_EQUALIZE, LUT_STRETCH = 0, 1
IMG_RAMP12, IMG_UNIFORM16 = 0, 1
MAT_EXACT8, MAT_UNIFORM32 = 0, 1
PREC_F32, PREC_TF32, PREC_BF16 = 0, 1, 2


class Stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("lo", C.c_uint32), ("hi", C.c_uint32), ("cdf_min", C.c_uint64)]


def build() -> None:
    """Builds the oracle (and the reference when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "-j8"], check=True)


def _load_orc() -> C.CDLL:
    if not ORC_PATH.exists():
        build()
    lib = C.CDLL(str(ORC_PATH))
    u64, vp, i32 = C.c_uint64, C.c_void_p, C.c_int
    sigs = {
        "orc_splitmix64": ([u64], u64),
        "orc_seed_b": ([u64], u64),
        "orc_synth_image": ([i32, u64, u64, u64, u64, u64, vp], None),
        "orc_synth_matrix": ([i32, u64, u64, u64, u64, u64, vp], None),
        "orc_lut_hist": ([vp, u64, vp, i32], None),
        "orc_lut_from_hist": ([vp, i32, vp, vp], i32),
        "orc_lut_gen": ([vp, u64, i32, vp, vp, i32], i32),
        "orc_lut_apply": ([vp, vp, vp, u64, i32], None),
        "orc_lut_correct": ([vp, vp, u64, i32, vp, vp, i32], i32),
        "orc_digest_u16": ([vp, u64, u64], u64),
        "orc_round_tf32": ([C.c_float], C.c_float),
        "orc_round_bf16": ([C.c_float], C.c_float),
        "orc_round_matrix": ([i32, vp, vp, u64, i32], None),
        "orc_matmul_f64": ([u64, u64, u64, vp, vp, vp, u64, vp, vp, i32], None),
        "orc_matmul_f32": ([u64, u64, u64, vp, vp, vp, i32], None),
        "orc_max_threads": ([], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


orc = _load_orc()


def _ptr(a: np.ndarray | None):
    return C.c_void_p(a.ctypes.data if a is not None else None)


def max_threads() -> int:
    return orc.orc_max_threads()


def synth_image(kind: int, seed: int, rows: int, cols: int, row0: int = 0, nrows: int | None = None) -> np.ndarray:
    nrows = rows - row0 if nrows is None else nrows
    out = np.empty(nrows * cols, dtype=np.uint16)
    orc.orc_synth_image(kind, seed, rows, cols, row0, nrows, _ptr(out))
    return out


def synth_matrix(kind: int, seed: int, rows: int, cols: int, row0: int = 0, nrows: int | None = None) -> np.ndarray:
    nrows = rows - row0 if nrows is None else nrows
    out = np.empty((nrows, cols), dtype=np.float32)
    orc.orc_synth_matrix(kind, seed, rows, cols, row0, nrows, _ptr(out))
    return out


def splitmix64(x: int) -> int:
    """The generators' hash, in Python: sample positions of
    header-only MATMUL requests."""
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def seed_b(seed: int) -> int:
    return orc.orc_seed_b(seed)


def lut_hist(img: np.ndarray, threads: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint16)
    hist = np.empty(65536, dtype=np.uint64)
    orc.orc_lut_hist(_ptr(img), img.size, _ptr(hist), threads)
    return hist


def lut_from_hist(hist: np.ndarray, mode: int) -> tuple[np.ndarray, dict]:
    hist = np.ascontiguousarray(hist, dtype=np.uint64)
    lut = np.empty(65536, dtype=np.uint16)
    st = Stats()
    rc = orc.orc_lut_from_hist(_ptr(hist), mode, _ptr(lut), C.byref(st))
    if rc != 0:
        return np.arange(65536, dtype=np.uint16), {"n": 0, "lo": 0, "hi": 0, "cdf_min": 0}
    return lut, {"n": st.n, "lo": st.lo, "hi": st.hi, "cdf_min": st.cdf_min}


def lut_gen(img: np.ndarray, mode: int, threads: int = 0) -> tuple[np.ndarray, dict]:
    return lut_from_hist(lut_hist(img, threads), mode)


def lut_apply(lut: np.ndarray, img: np.ndarray, threads: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint16)
    lut = np.ascontiguousarray(lut, dtype=np.uint16)
    out = np.empty_like(img)
    orc.orc_lut_apply(_ptr(lut), _ptr(img), _ptr(out), img.size, threads)
    return out


def lut_correct(img: np.ndarray, mode: int, threads: int = 0) -> tuple[np.ndarray, np.ndarray, dict]:
    img = np.ascontiguousarray(img, dtype=np.uint16)
    out = np.empty_like(img)
    lut = np.empty(65536, dtype=np.uint16)
    st = Stats()
    orc.orc_lut_correct(_ptr(img), _ptr(out), img.size, mode, _ptr(lut), C.byref(st), threads)
    return out, lut, {"n": st.n, "lo": st.lo, "hi": st.hi, "cdf_min": st.cdf_min}


def digest_u16(v: np.ndarray, index0: int = 0) -> int:
    v = np.ascontiguousarray(v, dtype=np.uint16)
    return orc.orc_digest_u16(_ptr(v), v.size, index0)


def round_matrix(prec: int, a: np.ndarray, threads: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty_like(a)
    orc.orc_round_matrix(prec, _ptr(a), _ptr(out), a.size, threads)
    return out


def matmul_f64(A: np.ndarray, B: np.ndarray, rows: np.ndarray | None = None, threads: int = 0):
    """(C, absprod) in f64 for the listed rows (all rows when None)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.uint64)
    nr = m if r is None else r.size
    Cm = np.empty((nr, n), dtype=np.float64)
    ab = np.empty((nr, n), dtype=np.float64)
    orc.orc_matmul_f64(m, n, k, _ptr(A), _ptr(B), _ptr(r), nr, _ptr(Cm), _ptr(ab), threads)
    return Cm, ab


def matmul_f32(A: np.ndarray, B: np.ndarray, threads: int = 0) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    m, k = A.shape
    _, n = B.shape
    Cm = np.empty((m, n), dtype=np.float32)
    orc.orc_matmul_f32(m, n, k, _ptr(A), _ptr(B), _ptr(Cm), threads)
    return Cm


# --------------------------------------------------------------------------
# The compiled reference (oracle/_ref/libgpc_ref.so)
# --------------------------------------------------------------------------

def _load_ref() -> C.CDLL | None:
    if not REF_PATH.exists():
        return None
    lib = C.CDLL(str(REF_PATH))
    u64, vp, i32, cp, sz = C.c_uint64, C.c_void_p, C.c_int, C.c_char_p, C.c_size_t
    sigs = {
        "ref_last_error": ([], cp),
        "ref_set_threads": ([i32], None),
        "ref_encode_header": ([cp, i32, cp, cp, vp], i32),
        "ref_decode_header": ([vp, sz, cp, C.POINTER(C.c_int), cp, cp], i32),
        "ref_params_roundtrip": ([cp, cp, sz], i32),
        "ref_params_get_uint": ([cp, cp, C.POINTER(C.c_uint64)], i32),
        "ref_expected_payload_len": ([cp, cp, C.POINTER(C.c_uint64)], i32),
        "ref_sanitize_message": ([cp, cp, cp, sz], i32),
        "ref_handle_request": ([vp, sz, vp, sz, C.POINTER(C.c_size_t)], i32),
        "ref_server_start": ([i32, i32, C.POINTER(vp), C.POINTER(C.c_uint16)], i32),
        "ref_server_stop": ([vp], i32),
        "ref_submit": ([cp, i32, cp, cp, vp, sz, cp, vp, sz, C.POINTER(C.c_size_t), cp, cp, cp], i32),
        "ref_demosaic": ([i32, i32, cp, sz, sz, vp, vp, i32], i32),
        "ref_normal_system": ([vp, vp, sz, i32, vp, vp], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


ref = _load_ref()


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"status {status}: {msg}")


def ref_check(st: int) -> None:
    if st != 0:
        raise RefError(st, ref.ref_last_error().decode(errors="replace"))


def ref_handle_request(request: bytes) -> bytes:
    cap = max(1 << 16, 4 * len(request) + 4096)
    buf = np.empty(cap, dtype=np.uint8)
    n = C.c_size_t(0)
    req = np.frombuffer(request, dtype=np.uint8) if request else np.zeros(1, np.uint8)
    st = ref.ref_handle_request(req.ctypes.data, len(request), buf.ctypes.data, cap, C.byref(n))
    if st == 24 and n.value > cap:  # SizeMismatch: retry with the size it needs
        buf = np.empty(n.value, dtype=np.uint8)
        st = ref.ref_handle_request(req.ctypes.data, len(request), buf.ctypes.data, n.value, C.byref(n))
    ref_check(st)
    return buf[: n.value].tobytes()


def ref_submit(port: int, flag: str, params: str, payload: bytes, name: str = "out.bin",
               resp_cap: int = 1 << 28, host: str = "127.0.0.1"):
    """Reference client::submit -> (status, params text, payload bytes, echoed name)."""
    buf = np.empty(resp_cap, dtype=np.uint8)
    n = C.c_size_t(0)
    status = C.create_string_buffer(64)
    rparams = C.create_string_buffer(256)
    rname = C.create_string_buffer(64)
    pl = np.frombuffer(payload, dtype=np.uint8) if payload else np.zeros(1, np.uint8)
    ref_check(ref.ref_submit(host.encode(), port, flag.encode(), params.encode(), pl.ctypes.data,
                             len(payload), name.encode(), buf.ctypes.data, resp_cap, C.byref(n),
                             status, rparams, rname))
    return status.value.decode(), rparams.value.decode(), buf[: n.value].tobytes(), rname.value.decode()


class RefServer:
    """The reference gpc server (builtins + oracle LUT/MATMUL descriptors)."""

    def __init__(self, max_tasks: int = 2):
        self.max_tasks = max_tasks
        self._h = C.c_void_p(None)
        self.port = 0

    def __enter__(self):
        bp = C.c_uint16(0)
        ref_check(ref.ref_server_start(0, self.max_tasks, C.byref(self._h), C.byref(bp)))
        self.port = bp.value
        return self

    def __exit__(self, *exc):
        ref_check(ref.ref_server_stop(self._h))


def ref_demosaic(gradient: bool, img: np.ndarray, rows: int, cols: int, phase: str = "RGGB",
                 gpcref: bool = False, workers: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint16)
    out = np.empty(3 * rows * cols, dtype=np.uint16)
    ref_check(ref.ref_demosaic(int(gradient), int(gpcref), phase.encode(), rows, cols,
                               img.ctypes.data, out.ctypes.data, workers))
    return out


def ref_normal_system(xs: np.ndarray, ys: np.ndarray, order: int) -> tuple[np.ndarray, np.ndarray]:
    """The reference's normal equations (gpc::lsq::build_normal_system,
    proj/src/lsq.cpp:69-90): A = V^T V ((order+1)^2, f64) and b = V^T y with
    V[i][j] = xs[i]^j -- contractions computed by the reference itself."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    m1 = order + 1
    a = np.empty((m1, m1), dtype=np.float64)
    b = np.empty(m1, dtype=np.float64)
    ref_check(ref.ref_normal_system(xs.ctypes.data, ys.ctypes.data, xs.size, order,
                                    a.ctypes.data, b.ctypes.data))
    return a, b


def host_cpu() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}
