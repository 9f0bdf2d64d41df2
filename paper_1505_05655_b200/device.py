"""Device-level calls on HBM-resident torch tensors (the C ABI's *_device
entry points).  torch supplies device memory and the stream; every byte of
compute happens in libgpcx.so's sm_100a kernels.

u16 images are carried in torch.int16 tensors (same bits; torch's uint16
support is partial) and compared as numpy uint16 views.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import IPC_HANDLE_BYTES, LutStats, check, lib

STATS_BYTES = C.sizeof(LutStats)


def _p(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else None)


def _s(stream: torch.cuda.Stream | None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def lut_workspace(n: int, device="cuda") -> torch.Tensor:
    nb = C.c_uint64(0)
    check(lib.gpcx_lut_workspace_size(n, C.byref(nb)))
    return torch.zeros(nb.value, dtype=torch.uint8, device=device)  # zeroed once


def new_lut(device="cuda") -> torch.Tensor:
    return torch.empty(65536, dtype=torch.int16, device=device)


def new_stats(device="cuda") -> torch.Tensor:
    return torch.zeros(STATS_BYTES, dtype=torch.uint8, device=device)


def read_stats(stats: torch.Tensor) -> dict[str, int]:
    raw = bytes(stats.cpu().numpy().tobytes())
    s = LutStats.from_buffer_copy(raw)
    return {"n": s.n, "lo": s.lo, "hi": s.hi, "cdf_min": s.cdf_min}


def lut_hist(img, hist, ws, stream=None):
    check(lib.gpcx_lut_hist_device(_p(img), img.numel(), _p(hist), _p(ws), ws.numel(), _s(stream)))


def lut_from_hist(hist, mode, lut, stats, ws, stream=None):
    check(lib.gpcx_lut_from_hist_device(_p(hist), mode, _p(lut), _p(stats), _p(ws), ws.numel(),
                                        _s(stream)))


def lut_correct_from_hist(hist, mode, inp, out, lut, stats, ws, stream=None):
    check(lib.gpcx_lut_correct_from_hist_device(_p(hist), mode, _p(inp), _p(out), inp.numel(),
                                                _p(lut), _p(stats), _p(ws), ws.numel(),
                                                _s(stream)))


def lut_minmax(img, stats, ws, stream=None):
    check(lib.gpcx_lut_minmax_device(_p(img), img.numel(), _p(stats), _p(ws), ws.numel(), _s(stream)))


def lut_from_minmax(stats, lut, stream=None):
    check(lib.gpcx_lut_from_minmax_device(_p(stats), _p(lut), _s(stream)))


def lut_gen(img, mode, lut, stats, ws, stream=None):
    check(lib.gpcx_lut_gen_device(_p(img), img.numel(), mode, _p(lut), _p(stats), _p(ws),
                                  ws.numel(), _s(stream)))


def lut_apply(lut, inp, out, stream=None):
    check(lib.gpcx_lut_apply_device(_p(lut), _p(inp), _p(out), inp.numel(), _s(stream)))


def lut_correct(inp, out, mode, lut, stats, ws, stream=None):
    check(lib.gpcx_lut_correct_device(_p(inp), _p(out), inp.numel(), mode, _p(lut), _p(stats),
                                      _p(ws), ws.numel(), _s(stream)))


class LutPeer:
    """One rank of a row-band LUT group whose histogram exchange runs inside
    the fused kernel over peer memory (gpcx_lut_peer_*, include/gpcx.h).

        p = LutPeer(rank, nranks)            # on the rank's current device
        handles = all_gather(p.handle())     # bytes, in rank order
        p.connect(handles)
        p.correct(band_in, band_out, mode, lut, stats, ws)   # every step
    """

    def __init__(self, rank: int, nranks: int):
        self._p = C.c_void_p(None)
        check(lib.gpcx_lut_peer_create(rank, nranks, C.byref(self._p)))
        self.rank, self.nranks = rank, nranks

    def handle(self) -> bytes:
        buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
        check(lib.gpcx_lut_peer_ipc_handle(self._p, buf))
        return bytes(buf)

    def connect(self, handles) -> None:
        blob = b"".join(handles)
        assert len(blob) == IPC_HANDLE_BYTES * self.nranks
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib.gpcx_lut_peer_connect(self._p, buf))

    def correct(self, inp, out, mode, lut, stats, ws, stream=None) -> None:
        check(lib.gpcx_lut_correct_peer_device(self._p, _p(inp), None if out is None else _p(out),
                                               inp.numel(), mode, _p(lut), _p(stats), _p(ws),
                                               ws.numel(), _s(stream)))

    def close(self) -> None:
        if self._p:
            check(lib.gpcx_lut_peer_destroy(self._p))
            self._p = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def matmul_workspace(prec: int, m: int, n: int, k: int, device="cuda") -> torch.Tensor | None:
    nb = C.c_uint64(0)
    check(lib.gpcx_matmul_workspace_size(prec, m, n, k, C.byref(nb)))
    return torch.empty(nb.value, dtype=torch.uint8, device=device) if nb.value else None


def matmul(prec, A, B, Cout, ws=None, stream=None):
    m, k = A.shape
    k2, n = B.shape
    assert k == k2 and tuple(Cout.shape) == (m, n)
    check(lib.gpcx_matmul_device(prec, m, n, k, _p(A), A.stride(0), _p(B), B.stride(0), _p(Cout),
                                 Cout.stride(0), _p(ws), ws.numel() if ws is not None else 0,
                                 _s(stream)))


def synth_image(kind, seed, rows, cols, row0=0, nrows=None, out=None, stream=None):
    nrows = rows - row0 if nrows is None else nrows
    if out is None:
        out = torch.empty(nrows * cols, dtype=torch.int16, device="cuda")
    check(lib.gpcx_synth_image_device(kind, seed, rows, cols, row0, nrows, _p(out), _s(stream)))
    return out


def synth_matrix(kind, seed, rows, cols, row0=0, nrows=None, out=None, stream=None):
    nrows = rows - row0 if nrows is None else nrows
    if out is None:
        out = torch.empty(nrows, cols, dtype=torch.float32, device="cuda")
    check(lib.gpcx_synth_matrix_device(kind, seed, rows, cols, row0, nrows, _p(out), _s(stream)))
    return out


def demosaic(gradient: bool, phase: int, mosaic, rows: int, cols: int, out=None, stream=None):
    """3 planes (R, G, B) of rows x cols u16 (int16 tensors) from a mosaic."""
    if out is None:
        out = torch.empty(3 * rows * cols, dtype=torch.int16, device=mosaic.device)
    check(lib.gpcx_demosaic_device(int(gradient), phase, _p(mosaic), _p(out), rows, cols, _s(stream)))
    return out


def digest_u16(v, index0=0, out=None, stream=None) -> torch.Tensor:
    if out is None:
        out = torch.zeros(1, dtype=torch.int64, device=v.device)
    check(lib.gpcx_digest_u16_device(_p(v), v.numel(), index0, _p(out), _s(stream)))
    return out
