"""Row-band / block-row shard planning across ranks (one process per GPU,
torch.distributed for the plumbing) -- SURVEY.md §8e.

  LUT_CORRECT : rank r owns rows band(rows, N, r); the one exchange is an
                all-reduce (sum) of the 65536-bin histogram (equalize) or of
                (min, max) (stretch); every rank then builds the identical
                LUT and applies it to its band.  The output stays sharded
                (each band in its GPU's HBM) or is gathered to rank 0.
  MATMUL      : rank r owns block rows band(m, N, r) of A and C and the
                k-slice band(k, N, r) of B; B is replicated (all-gather of
                the slices); no other exchange until the optional gather.

The compute steps are injected (`hist`, `lut_from_hist`, `apply`), so the
same exchange logic runs with the sm_100a kernels in bench.py and with the
CPU oracle over gloo in tests/test_shard.py.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


def band(rows: int, n: int, r: int) -> tuple[int, int]:
    """(first row, row count) of rank r's band: ceil(rows / n) rows each,
    the last band ragged; empty bands past the end."""
    per = (rows + n - 1) // n
    r0 = min(rows, r * per)
    return r0, min(per, rows - r0)


def bands(rows: int, n: int) -> list[tuple[int, int]]:
    return [band(rows, n, r) for r in range(n)]


@dataclass
class ShardedLut:
    """One LUT_CORRECT over row bands.  `dist` is torch.distributed (or None
    for a single rank); hist/lut/apply are the per-band compute steps."""

    dist: object | None
    hist: Callable       # band -> hist tensor (int32/int64, 65536)
    lut_from_hist: Callable  # global hist -> (lut, stats)
    apply: Callable      # (lut, band) -> corrected band

    def run(self, band_img):
        h = self.hist(band_img)
        if self.dist is not None and self.dist.is_initialized() and self.dist.get_world_size() > 1:
            self.dist.all_reduce(h)  # the only exchange step
        lut, stats = self.lut_from_hist(h)
        return self.apply(lut, band_img), lut, stats


def _bytes(t):
    """Byte view of a contiguous tensor (every backend carries u8; gloo has
    no int16)."""
    import torch
    return t.reshape(-1).view(torch.uint8)


def gather_bands(dist, band_out, rows_per_rank: list[int], cols: int):
    """Gathers every rank's band to rank 0 (the full image / matrix there,
    None elsewhere).  Exact sizes, no padding: rank 0 receives each band
    straight into its slice of the result (point-to-point, so ragged bands
    cost nothing extra)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return band_out
    world, rank = dist.get_world_size(), dist.get_rank()
    offs = [0]
    for r in rows_per_rank:
        offs.append(offs[-1] + r * cols)
    if rank != 0:
        if band_out.numel() > 0:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, _bytes(band_out), 0)]):
                w.wait()
        return None
    full = torch.empty(offs[-1], dtype=band_out.dtype, device=band_out.device)
    full[: band_out.numel()] = band_out.reshape(-1)
    ops = [dist.P2POp(dist.irecv, _bytes(full[offs[r]:offs[r + 1]]), r)
           for r in range(1, world) if offs[r + 1] > offs[r]]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return full


def replicate_rows(dist, own_rows, rows_per_rank: list[int], cols: int, out=None):
    """B replication for block-row MATMUL: rank r holds rows
    [sum(rows_per_rank[:r]), +rows_per_rank[r]) of B (its 1/N k-slice, staged
    over its own PCIe link or generated in place); afterwards every rank
    holds all of B in `out`.  Equal slices: one all-gather straight into
    `out`; ragged ones: one broadcast per owner into its rows of `out`.
    Device tensors over NCCL; over gloo (CPU plumbing) through host copies."""
    import torch
    total = sum(rows_per_rank)
    if out is None:
        out = torch.empty(total, cols, dtype=own_rows.dtype, device=own_rows.device)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        if out.data_ptr() != own_rows.data_ptr():
            out.copy_(own_rows.reshape(total, cols))
        return out
    rank = dist.get_rank()
    nccl = dist.get_backend() == "nccl"
    starts = [sum(rows_per_rank[:r]) for r in range(len(rows_per_rank))]
    dst = out if nccl or out.device.type == "cpu" else torch.empty(out.shape, dtype=out.dtype)
    src = own_rows if nccl or own_rows.device.type == "cpu" else own_rows.cpu()
    if len(set(rows_per_rank)) == 1 and nccl:
        dist.all_gather_into_tensor(_bytes(dst), _bytes(src))
    elif len(set(rows_per_rank)) == 1:
        dist.all_gather(list(_bytes(dst).chunk(len(rows_per_rank))), _bytes(src))
    else:
        dst[starts[rank]:starts[rank] + rows_per_rank[rank]].copy_(src.reshape(-1, cols))
        for r, n in enumerate(rows_per_rank):
            if n:
                dist.broadcast(_bytes(dst[starts[r]:starts[r] + n]), src=r)
    if dst is not out:
        out.copy_(dst)
    return out


@dataclass
class ShardedMatmul:
    """One MATMUL over block rows: rank r owns rows band(m, N, r) of A and C
    and the k-slice band(k, N, r) of B's rows; B is replicated (the path's
    one exchange), then each rank multiplies its rows.  The tile / K order
    of the kernel does not depend on N, so C is bitwise identical for any
    rank count (the analogue of proj/tests/acceptance.cpp:278-315)."""

    dist: object | None
    matmul: Callable     # (A band, full B) -> C band

    def run(self, a_band, b_slice, k: int, n: int, world: int):
        B = replicate_rows(self.dist, b_slice, [band(k, world, r)[1] for r in range(world)], n)
        return self.matmul(a_band, B)
