"""ctypes binding of include/gpcx.h (libgpcx.so).

The library is the product: there is no Python or CPU fallback.  If the
shared library is missing this module raises at import time; if no GPU is
usable, every compute call fails with GPCX_E_TASK_FAILED (-> GpcxError).
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from pathlib import Path

# GPCX_LIB_PATH selects another build of the same library (the
# ThreadSanitizer build, tools/tsan_server.sh); the default is the product.
LIB_PATH = Path(os.environ.get("GPCX_LIB_PATH") or
                Path(__file__).resolve().parent / "lib" / "libgpcx.so")

OK = 0
ERRC_NAMES = [
    "FieldTooLong", "InvalidCharacter", "BadMarker", "MalformedPadding", "DuplicateKey",
    "BadToken", "MissingParam", "BadValue", "Overflow", "Truncated", "PayloadMismatch",
    "UnknownTask", "DuplicateFlag", "TaskFailed", "BadImage", "InsufficientPoints", "Singular",
    "OrderTooHigh", "ConnectFailed", "BindFailed", "TimedOut", "IoError", "UnsafeName",
    "SizeMismatch", "BadFormat", "TooLarge", "ServerError",
]
STATUS = {name: i + 1 for i, name in enumerate(ERRC_NAMES)}

LUT_EQUALIZE, LUT_STRETCH = 0, 1
IMG_RAMP12, IMG_UNIFORM16 = 0, 1
MAT_EXACT8, MAT_UNIFORM32 = 0, 1
PREC_F32, PREC_TF32, PREC_BF16 = 0, 1, 2
OP_LUT_GEN, OP_LUT_APPLY, OP_LUT_CORRECT = 0, 1, 2
PREC_BY_NAME = {"f32": PREC_F32, "tf32": PREC_TF32, "bf16": PREC_BF16}
MODE_BY_NAME = {"equalize": LUT_EQUALIZE, "stretch": LUT_STRETCH}

# Every symbol include/gpcx.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "gpcx_abi_version", "gpcx_init", "gpcx_shutdown", "gpcx_device_count", "gpcx_last_error",
    "gpcx_status_name", "gpcx_response_code", "gpcx_payload_len", "gpcx_output_len",
    "gpcx_required_params", "gpcx_flags", "gpcx_run", "gpcx_lut_host", "gpcx_matmul_host",
    "gpcx_pinned_alloc", "gpcx_pinned_free",
    "gpcx_lut_workspace_size", "gpcx_lut_hist_device", "gpcx_lut_from_hist_device",
    "gpcx_lut_correct_from_hist_device",
    "gpcx_lut_minmax_device", "gpcx_lut_from_minmax_device", "gpcx_lut_gen_device",
    "gpcx_lut_apply_device", "gpcx_lut_correct_device", "gpcx_matmul_workspace_size",
    "gpcx_matmul_device", "gpcx_synth_image_device", "gpcx_synth_matrix_device",
    "gpcx_digest_u16_device", "gpcx_server_start", "gpcx_server_stop", "gpcx_handle_request",
    "gpcx_demosaic_device", "gpcx_devinfo_probe", "gpcx_devinfo_render", "gpcx_client_submit",
    "gpcx_lut_peer_create", "gpcx_lut_peer_ipc_handle", "gpcx_lut_peer_connect",
    "gpcx_lut_peer_destroy", "gpcx_lut_correct_peer_device", "gpcx_server_stats_get",
    "gpcx_device_health", "gpcx_debug_fault",
]
IPC_HANDLE_BYTES = 64

PHASES = {"RGGB": 0, "BGGR": 1, "GRBG": 2, "GBRG": 3}


class DeviceInfo(C.Structure):
    _fields_ = [("name", C.c_char * 256), ("compute_capability", C.c_char * 16),
                ("warp_size", C.c_int32), ("total_constant_memory", C.c_uint64),
                ("total_global_memory", C.c_uint64), ("shared_memory_per_block", C.c_uint64),
                ("clock_rate_khz", C.c_int64), ("multi_processor_count", C.c_int32),
                ("registers_per_block", C.c_int32), ("max_threads_per_block", C.c_int32),
                ("max_grid_size", C.c_int32 * 3), ("max_threads_dim", C.c_int32 * 3)]


class ServerStats(C.Structure):
    _fields_ = [("requests", C.c_uint64), ("recv_ms", C.c_double), ("task_ms", C.c_double),
                ("send_ms", C.c_double), ("busy", C.c_uint64), ("dropped", C.c_uint64)]


class LutStats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("lo", C.c_uint32), ("hi", C.c_uint32), ("cdf_min", C.c_uint64)]


class GpcxError(RuntimeError):
    """A non-zero gpcx_status; .code is the gpc::Errc name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERRC_NAMES[status - 1] if 1 <= status <= len(ERRC_NAMES) else "Unknown"
        super().__init__(f"{self.code}: {message}")


def _building() -> bool:
    """`python -m paper_1505_05655_b200.build`: Python imports this package
    (and so this module) before it runs build.py, so a clean checkout must
    not fail here -- the library is built first, then loaded."""
    argv = list(getattr(sys, "orig_argv", []))
    return "-m" in argv and argv[argv.index("-m") + 1:argv.index("-m") + 2] == [f"{__package__}.build"]


def _load() -> C.CDLL:
    if not LIB_PATH.exists() and _building():
        import runpy
        runpy.run_path(str(LIB_PATH.parent.parent / "build.py"), run_name="build_only")["build"]()
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1505_05655_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    u64, u32, vp, cp, i32 = C.c_uint64, C.c_uint32, C.c_void_p, C.c_char_p, C.c_int
    pu64 = C.POINTER(C.c_uint64)
    sig = {
        "gpcx_abi_version": ([], i32),
        "gpcx_init": ([i32, C.POINTER(C.c_int)], i32),
        "gpcx_shutdown": ([], i32),
        "gpcx_device_count": ([C.POINTER(C.c_int)], i32),
        "gpcx_last_error": ([], cp),
        "gpcx_status_name": ([i32], cp),
        "gpcx_response_code": ([i32], cp),
        "gpcx_payload_len": ([cp, cp, pu64], i32),
        "gpcx_output_len": ([cp, cp, pu64], i32),
        "gpcx_required_params": ([cp, cp, u64], i32),
        "gpcx_flags": ([cp, u64], i32),
        "gpcx_run": ([cp, cp, vp, u64, vp, u64, pu64, cp, u64], i32),
        "gpcx_lut_host": ([i32, i32, u64, u64, vp, vp, vp, vp, vp], i32),
        "gpcx_matmul_host": ([i32, u64, u64, u64, vp, vp, vp], i32),
        "gpcx_pinned_alloc": ([u64], vp),
        "gpcx_pinned_free": ([vp], None),
        "gpcx_lut_workspace_size": ([u64, pu64], i32),
        "gpcx_lut_hist_device": ([vp, u64, vp, vp, u64, vp], i32),
        "gpcx_lut_from_hist_device": ([vp, i32, vp, vp, vp, u64, vp], i32),
        "gpcx_lut_correct_from_hist_device": ([vp, i32, vp, vp, u64, vp, vp, vp, u64, vp], i32),
        "gpcx_lut_minmax_device": ([vp, u64, vp, vp, u64, vp], i32),
        "gpcx_lut_from_minmax_device": ([vp, vp, vp], i32),
        "gpcx_lut_gen_device": ([vp, u64, i32, vp, vp, vp, u64, vp], i32),
        "gpcx_lut_apply_device": ([vp, vp, vp, u64, vp], i32),
        "gpcx_lut_correct_device": ([vp, vp, u64, i32, vp, vp, vp, u64, vp], i32),
        "gpcx_matmul_workspace_size": ([i32, u64, u64, u64, pu64], i32),
        "gpcx_matmul_device": ([i32, u64, u64, u64, vp, u64, vp, u64, vp, u64, vp, u64, vp], i32),
        "gpcx_synth_image_device": ([i32, u64, u64, u64, u64, u64, vp, vp], i32),
        "gpcx_synth_matrix_device": ([i32, u64, u64, u64, u64, u64, vp, vp], i32),
        "gpcx_digest_u16_device": ([vp, u64, u64, vp, vp], i32),
        "gpcx_server_start": ([cp, C.c_uint16, i32, i32, C.POINTER(vp), C.POINTER(C.c_uint16)], i32),
        "gpcx_server_stop": ([vp], i32),
        "gpcx_handle_request": ([vp, u64, vp, u64, pu64], i32),
        "gpcx_demosaic_device": ([i32, i32, vp, vp, u64, u64, vp], i32),
        "gpcx_devinfo_probe": ([vp, i32, C.POINTER(C.c_int)], i32),
        "gpcx_devinfo_render": ([vp, i32, cp, u64, pu64], i32),
        "gpcx_client_submit": ([cp, C.c_uint16, cp, cp, C.POINTER(vp), pu64, i32, cp, vp, u64, pu64,
                                cp, u64, cp, u64], i32),
        "gpcx_lut_peer_create": ([i32, i32, C.POINTER(vp)], i32),
        "gpcx_lut_peer_ipc_handle": ([vp, vp], i32),
        "gpcx_lut_peer_connect": ([vp, vp], i32),
        "gpcx_lut_peer_destroy": ([vp], i32),
        "gpcx_lut_correct_peer_device": ([vp, vp, vp, u64, i32, vp, vp, vp, u64, vp], i32),
        "gpcx_server_stats_get": ([vp, vp], i32),
        "gpcx_device_health": ([i32, C.POINTER(C.c_int), cp, u64], i32),
        "gpcx_debug_fault": ([i32, i32], i32),
    }
    assert set(sig) == set(EXPORTS)
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(status: int) -> None:
    if status != OK:
        raise GpcxError(status, lib.gpcx_last_error().decode(errors="replace"))
