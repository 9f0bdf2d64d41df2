"""paper_1505_05655_b200 -- B200-native task backend for the remote-GPGPU
task server of arXiv:1505.05655 (reference: `gpc`, /root/reference).

The product is the C++/CUDA library libgpcx.so (include/gpcx.h): sm_100a
kernels for LUT_GEN / LUT_APPLY / LUT_CORRECT / MATMUL, the pinned-staging
task executor and the TCP server that speaks the reference's 260-byte wire
format.  This package is a thin ctypes layer over it for tests, bench.py and
Python callers; it never computes anything itself.
"""
from __future__ import annotations

import ctypes as C
from typing import Mapping

import numpy as np

from ._lib import (  # noqa: F401
    EXPORTS, PHASES, DeviceInfo, GpcxError, IMG_RAMP12, IMG_UNIFORM16, LIB_PATH, LUT_EQUALIZE,
    LUT_STRETCH, LutStats, ServerStats, MAT_EXACT8, MAT_UNIFORM32, MODE_BY_NAME, PREC_BF16, PREC_BY_NAME,
    PREC_F32, PREC_TF32, STATUS, check, lib,
)


def devinfo_probe() -> list[DeviceInfo]:
    arr = (DeviceInfo * 64)()
    n = C.c_int(0)
    check(lib.gpcx_devinfo_probe(arr, 64, C.byref(n)))
    return list(arr[: min(n.value, 64)])


def devinfo_render(devices: list[DeviceInfo]) -> str:
    arr = (DeviceInfo * max(1, len(devices)))(*devices)
    need = C.c_uint64(0)
    lib.gpcx_devinfo_render(arr, len(devices), None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value + 1)
    check(lib.gpcx_devinfo_render(arr, len(devices), buf, need.value + 1, C.byref(need)))
    return buf.value.decode()

__all__ = [
    "GpcxError", "init", "shutdown", "device_count", "run", "payload_len", "output_len",
    "params_text", "parse_params", "Server", "handle_request", "flags", "required_params",
    "device_health",
]


def params_text(params: str | Mapping[str, object] | None) -> str:
    """Params slot text: k=v joined by ',' (values' ',' folded to ';')."""
    if params is None:
        return ""
    if isinstance(params, str):
        return params
    return ",".join(f"{k}={str(v).replace(',', ';')}" for k, v in params.items())


def parse_params(text: str) -> dict[str, str]:
    out: dict[str, str] = {}
    if not text:
        return out
    for tok in text.split(","):
        k, _, v = tok.partition("=")
        out[k] = v.replace(";", ",")
    return out


def init(devices: list[int] | None = None) -> None:
    devs = list(devices or [])
    arr = (C.c_int * max(1, len(devs)))(*devs) if devs else None
    check(lib.gpcx_init(len(devs), arr))


def shutdown() -> None:
    check(lib.gpcx_shutdown())


def device_count() -> int:
    n = C.c_int(0)
    check(lib.gpcx_device_count(C.byref(n)))
    return n.value


def device_health(index: int) -> tuple[bool, str]:
    """(healthy, reason) of bound device `index` (gpcx_device_health)."""
    ok = C.c_int(0)
    why = C.create_string_buffer(512)
    check(lib.gpcx_device_health(index, C.byref(ok), why, 512))
    return bool(ok.value), why.value.decode(errors="replace")


def flags() -> list[str]:
    buf = C.create_string_buffer(256)
    check(lib.gpcx_flags(buf, 256))
    return buf.value.decode().split(",")


def required_params(flag: str) -> list[str]:
    buf = C.create_string_buffer(256)
    check(lib.gpcx_required_params(flag.encode(), buf, 256))
    return [p for p in buf.value.decode().split(",") if p]


def payload_len(flag: str, params) -> int:
    n = C.c_uint64(0)
    check(lib.gpcx_payload_len(flag.encode(), params_text(params).encode(), C.byref(n)))
    return n.value


def output_len(flag: str, params) -> int:
    n = C.c_uint64(0)
    check(lib.gpcx_output_len(flag.encode(), params_text(params).encode(), C.byref(n)))
    return n.value


def _host_ptr(payload) -> tuple[int, int, object]:
    if payload is None:
        return 0, 0, None
    if isinstance(payload, (bytes, bytearray)):
        arr = np.frombuffer(payload, dtype=np.uint8)
    else:
        arr = np.ascontiguousarray(payload)
    return arr.ctypes.data, arr.nbytes, arr


def run(flag: str, params, payload, out: np.ndarray | None = None) -> tuple[dict[str, str], np.ndarray]:
    """gpcx_run: one task request through the C ABI with host buffers.

    Returns (result params, response payload as a uint8 array)."""
    text = params_text(params)
    want = output_len(flag, text)
    if out is None:
        out = np.empty(want, dtype=np.uint8)
    ptr, nbytes, keep = _host_ptr(payload)
    got = C.c_uint64(0)
    rp = C.create_string_buffer(512)
    check(lib.gpcx_run(flag.encode(), text.encode(), C.c_void_p(ptr), nbytes,
                       C.c_void_p(out.ctypes.data), out.nbytes, C.byref(got), rp, 512))
    del keep
    return parse_params(rp.value.decode()), out.view(np.uint8)[: got.value]


def handle_request(request: bytes) -> bytes:
    """Serve one in-memory request frame (srv::handle_connection)."""
    cap = C.c_uint64(0)
    buf = (C.c_uint8 * 4096)()
    req = np.frombuffer(request, dtype=np.uint8) if request else np.zeros(1, np.uint8)
    st = lib.gpcx_handle_request(C.c_void_p(req.ctypes.data), len(request), buf, 4096, C.byref(cap))
    if st == STATUS["SizeMismatch"] and cap.value > 4096:
        big = np.empty(cap.value, dtype=np.uint8)
        st = lib.gpcx_handle_request(C.c_void_p(req.ctypes.data), len(request),
                                     C.c_void_p(big.ctypes.data), cap.value, C.byref(cap))
        check(st)
        return big.tobytes()
    check(st)
    return bytes(buf[: cap.value])


class Server:
    """The B200 task server (gpcx_server_start / gpcx_server_stop)."""

    def __init__(self, bind: str = "127.0.0.1", port: int = 0, max_tasks: int = 2,
                 idle_timeout_ms: int = 30000):
        self._args = (bind, port, max_tasks, idle_timeout_ms)
        self._h = C.c_void_p(None)
        self.port = 0

    def start(self) -> "Server":
        bind, port, max_tasks, idle = self._args
        bp = C.c_uint16(0)
        check(lib.gpcx_server_start(bind.encode(), port, max_tasks, idle, C.byref(self._h), C.byref(bp)))
        self.port = bp.value
        return self

    def stop(self) -> None:
        if self._h.value:
            check(lib.gpcx_server_stop(self._h))
            self._h = C.c_void_p(None)

    def stats(self) -> dict:
        """Cumulative phase times (ms, summed) of the answered requests."""
        st = ServerStats()
        check(lib.gpcx_server_stats_get(self._h, C.byref(st)))
        return {"requests": st.requests, "recv_ms": st.recv_ms, "task_ms": st.task_ms,
                "send_ms": st.send_ms, "busy": st.busy, "dropped": st.dropped}

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()
