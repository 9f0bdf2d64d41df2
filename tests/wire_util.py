"""Byte-level helpers for request frames (the 260-byte header of
proj/include/gpc/wire.hpp:15-47) -- a third, test-only encoder so the
tests can build malformed frames the C++ encoders refuse to produce."""
from __future__ import annotations

import random
import socket

HEADER = 260
MARK_DATA, MARK_NONE = 0x2B, 0x00


def header(flag: str, params: str = "", name: str = "out.bin", marker: int | None = None,
           has_payload: bool = False) -> bytes:
    h = bytearray(HEADER)
    fb, pb, nb = flag.encode("latin1"), params.encode("latin1"), name.encode("latin1")
    h[0:len(fb)] = fb[:29]
    h[29] = (MARK_DATA if has_payload else MARK_NONE) if marker is None else marker
    h[30:30 + len(pb)] = pb[:200]
    h[230:230 + len(nb)] = nb[:30]
    return bytes(h)


def frame(flag: str, params: str, payload: bytes = b"", name: str = "out.bin") -> bytes:
    return header(flag, params, name, has_payload=bool(payload)) + payload


def parse_response(resp: bytes) -> dict:
    assert len(resp) >= HEADER, len(resp)
    h = resp[:HEADER]

    def slot(a, b):
        return h[a:b].split(b"\0", 1)[0].decode("latin1")

    return {"status": slot(0, 29), "marker": h[29], "params": slot(30, 230),
            "name": slot(230, 260), "payload": resp[HEADER:]}


def printable(rng: random.Random, n: int) -> str:
    return "".join(chr(rng.randint(0x20, 0x7E)) for _ in range(rng.randint(0, n)))


def roundtrip(port: int, data: bytes, host: str = "127.0.0.1", timeout: float = 30.0) -> bytes:
    """Sends raw bytes, half-closes, reads the whole response."""
    with socket.create_connection((host, port), timeout=timeout) as s:
        s.sendall(data)
        s.shutdown(socket.SHUT_WR)
        chunks = []
        while True:
            b = s.recv(1 << 20)
            if not b:
                break
            chunks.append(b)
    return b"".join(chunks)
