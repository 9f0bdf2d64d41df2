"""Row-band / block-row shard planning across ranks (one process per GPU,
torch.distributed for the plumbing) -- SURVEY.md §8e.

  LUT_CORRECT : rank r owns rows band(rows, N, r); the one exchange is an
                all-reduce (sum) of the 65536-bin histogram (equalize) or of
                (min, max) (stretch); every rank then builds the identical
                LUT and applies it to its band.  The output stays sharded
                (each band in its GPU's HBM) or is gathered to rank 0.
  MATMUL      : rank r owns block rows band(m, N, r) of A and C; B is
                replicated; no exchange until the optional gather.

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


def gather_bands(dist, band_out, rows_per_rank: list[int], cols: int):
    """Gathers every rank's band to rank 0 (returns the full image there,
    None elsewhere); bands may be ragged."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return band_out
    world = dist.get_world_size()
    per = max(rows_per_rank)
    padded = torch.zeros(per * cols, dtype=band_out.dtype, device=band_out.device)
    padded[: band_out.numel()] = band_out.reshape(-1)
    wire = padded.view(torch.uint8)  # bytes: every backend carries u8 (gloo has no int16)
    parts = [torch.empty_like(wire) for _ in range(world)] if dist.get_rank() == 0 else None
    dist.gather(wire, parts, dst=0)
    if dist.get_rank() != 0:
        return None
    return torch.cat([p.view(band_out.dtype)[: r * cols] for p, r in zip(parts, rows_per_rank)])
