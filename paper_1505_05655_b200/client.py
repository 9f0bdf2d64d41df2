"""Minimal Python client of the task server's wire protocol -- the same
260-byte header and framing as the reference client::submit
(proj/src/client.cpp:97-129): one request per connection, the response
payload sized by its bytes= param, an ERR status returned as data.
"""
from __future__ import annotations

import socket
from dataclasses import dataclass

HEADER = 260


@dataclass
class TaskResult:
    status: str
    params: dict
    payload: bytearray
    output_name: str

    @property
    def ok(self) -> bool:
        return self.status == "OK"


def _slot(text: str, size: int) -> bytes:
    b = text.encode("ascii")
    if len(b) > size or any(c < 0x20 or c > 0x7E for c in b):
        raise ValueError(f"field does not fit its {size}-byte slot: {text!r}")
    return b + b"\0" * (size - len(b))


def encode_header(flag: str, params: str, output_name: str, has_payload: bool) -> bytes:
    return (_slot(flag, 29) + (b"\x2b" if has_payload else b"\x00") + _slot(params, 200)
            + _slot(output_name, 30))


def _params_text(params) -> str:
    if isinstance(params, str):
        return params
    return ",".join(f"{k}={str(v).replace(',', ';')}" for k, v in params.items())


def _recv_exact(s: socket.socket, n: int) -> bytearray:
    buf = bytearray(n)
    view = memoryview(buf)
    got = 0
    while got < n:
        k = s.recv_into(view[got:], n - got)
        if k == 0:
            raise ConnectionError(f"truncated response: got {got} of {n} bytes")
        got += k
    return buf


def submit_native(host: str, port: int, flag: str, params, parts=(), resp_cap: int = 0,
                  output_name: str = "", out=None) -> TaskResult:
    """The same request through libgpcx's C++ client (gpcx_client_submit):
    socket I/O off the GIL, payload parts sent without concatenation, the
    response written into `out` (a writable buffer of >= resp_cap bytes) or
    a new bytearray."""
    import ctypes as C

    import numpy as np

    from ._lib import check, lib
    text = _params_text(params)
    arrays = [np.frombuffer(memoryview(p).cast("B"), dtype=np.uint8) for p in parts]
    ptrs = (C.c_void_p * max(1, len(arrays)))(*[a.ctypes.data for a in arrays])
    lens = (C.c_uint64 * max(1, len(arrays)))(*[a.nbytes for a in arrays])
    if out is None:
        out = bytearray(resp_cap)
    ob = (C.c_char * len(out)).from_buffer(out) if len(out) else None
    got = C.c_uint64(0)
    status = C.create_string_buffer(64)
    rparams = C.create_string_buffer(256)
    check(lib.gpcx_client_submit(host.encode(), port, flag.encode(), text.encode(), ptrs, lens,
                                 len(arrays), output_name.encode(), ob, len(out), C.byref(got),
                                 status, 64, rparams, 256))
    params_out = {}
    for tok in filter(None, rparams.value.decode().split(",")):
        k, _, v = tok.partition("=")
        params_out[k] = v.replace(";", ",")
    return TaskResult(status.value.decode(), params_out, memoryview(out)[: got.value], output_name)


def submit(host: str, port: int, flag: str, params, payload=b"",
           output_name: str = "", timeout: float = 300.0) -> TaskResult:
    """`payload` is bytes-like or a list of bytes-like parts sent back to
    back (e.g. LUT || image without concatenating them)."""
    text = _params_text(params)
    parts = payload if isinstance(payload, (list, tuple)) else [payload]
    parts = [memoryview(p).cast("B") for p in parts if len(memoryview(p).cast("B"))]
    with socket.create_connection((host, port), timeout=timeout) as s:
        s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        s.sendall(encode_header(flag, text, output_name, bool(parts)))
        for p in parts:
            s.sendall(p)
        head = _recv_exact(s, HEADER)
        status = head[:29].split(b"\0", 1)[0].decode()
        ptext = head[30:230].split(b"\0", 1)[0].decode()
        name = head[230:260].split(b"\0", 1)[0].decode()
        params_out = {}
        for tok in filter(None, ptext.split(",")):
            k, _, v = tok.partition("=")
            params_out[k] = v.replace(";", ",")
        n = int(params_out.get("bytes", "0")) if head[29] == 0x2B else 0
        body = _recv_exact(s, n) if n else bytearray()
    return TaskResult(status, params_out, body, name)
