"""The N>1 path on CPU: world_size 2 (and 3) over gloo, one process per
rank, running paper_1505_05655_b200.shard's exchange logic with the CPU
oracle as the per-band compute.  The sharded result must equal the
single-process oracle bit-for-bit (the parexec invariance contract carried
to ranks)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_05655_b200.shard import ShardedLut, band, bands, gather_bands

ROOT = Path(__file__).resolve().parent.parent


def test_band_partition_covers_rows_once():
    for rows in (1, 2, 7, 32768, 4099):
        for n in (1, 2, 3, 4, 8):
            bs = bands(rows, n)
            covered = [r for r0, nr in bs for r in range(r0, r0 + nr)]
            assert covered == list(range(rows))
            assert band(rows, n, n - 1)[0] + band(rows, n, n - 1)[1] <= rows


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows, cols, mode, q):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, nr = band(rows, world, rank)
    img = torch.from_numpy(O.synth_image(O.IMG_UNIFORM16 if mode else O.IMG_RAMP12, 7, rows, cols, r0, nr)
                           .astype(np.int64))

    def hist(b):
        return torch.from_numpy(O.lut_hist(b.numpy().astype(np.uint16)).astype(np.int64))

    def lut_from_hist(h):
        return O.lut_from_hist(h.numpy().astype(np.uint64), mode)

    def apply(lut, b):  # int16 carrier, like the device path (gather moves bytes)
        return torch.from_numpy(lut[b.numpy()].astype(np.uint16).view(np.int16))

    out, lut, stats = ShardedLut(dist, hist, lut_from_hist, apply).run(img)
    full = gather_bands(dist, out, [nr_ for _, nr_ in bands(rows, world)], cols)
    if rank == 0:
        q.put((full.numpy().astype(np.uint16).tobytes(), lut.tobytes(), stats))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, 0), (2, 1), (3, 0)])
def test_sharded_lut_correct_over_gloo_equals_single_process(world, mode):
    from oracle import oracle as O
    rows, cols = 301, 173  # ragged bands
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, mode, q)) for r in range(world)]
    [p.start() for p in procs]
    out, lut, stats = q.get(timeout=120)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    img = O.synth_image(O.IMG_UNIFORM16 if mode else O.IMG_RAMP12, 7, rows, cols)
    r_out, r_lut, r_st = O.lut_correct(img, mode)
    assert out == r_out.tobytes()
    assert lut == r_lut.tobytes()
    assert stats == r_st


class _FakePeer:
    def __init__(self, rank, fail_at):
        self.rank, self.fail_at, self.closed, self.connected = rank, fail_at, False, None
        if fail_at == ("create", rank):
            raise RuntimeError("no device block")

    def handle(self):
        return bytes([self.rank]) * 64

    def connect(self, handles):
        if self.fail_at == ("connect", self.rank):
            raise RuntimeError("no P2P path")
        self.connected = handles

    def close(self):
        self.closed = True


def _negotiate_worker(rank, world, port, fail_at, q):
    sys.path.insert(0, str(ROOT))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank))
    d = bench.Dist(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d.pg = dist  # (Dist.init would bind a CUDA device)
    peer = bench.open_peer_exchange(d, lambda: _FakePeer(rank, fail_at), "cpu")
    q.put((rank, None if peer is None else [h[0] for h in peer.connected]))
    d.close()


@pytest.mark.parametrize("fail_at", [None, ("create", 1), ("connect", 0)])
def test_peer_exchange_negotiation_is_unanimous(fail_at):
    """bench.open_peer_exchange: every rank connects with all handles in
    rank order, or -- if any rank cannot create or connect its block --
    every rank falls back to the NCCL exchange (no rank left waiting)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_negotiate_worker, args=(world, port, fail_at, q), nprocs=world,
                       start_method="spawn", join=True)
    got = dict(q.get(timeout=60) for _ in range(world))
    if fail_at is None:
        assert got == {0: [0, 1], 1: [0, 1]}
    else:
        assert got == {0: None, 1: None}


def _mm_worker(rank, world, port, m, k, n, q):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    from paper_1505_05655_b200.shard import ShardedMatmul
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, nr = band(m, world, rank)
    k0, nk = band(k, world, rank)
    a = torch.from_numpy(O.synth_matrix(O.MAT_UNIFORM32, 9, m, k, r0, nr))
    b = torch.from_numpy(O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(9), k, n, k0, nk))
    c = ShardedMatmul(dist, lambda A, B: torch.from_numpy(O.matmul_f32(A.numpy(), B.numpy()))).run(
        a, b, k, n, world)
    full = gather_bands(dist, c, [nr_ for _, nr_ in bands(m, world)], n)
    if rank == 0:
        q.put(full.numpy().tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,k,n", [(2, 64, 96, 40), (3, 67, 101, 33)])
def test_sharded_matmul_over_gloo_equals_single_process(world, m, k, n):
    """Block rows of A / C per rank, B replicated from per-rank k-slices
    (equal slices: all-gather; ragged: per-owner broadcasts), C gathered
    with exact sizes: bitwise equal to the single-process product."""
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mm_worker, args=(r, world, port, m, k, n, q)) for r in range(world)]
    [p.start() for p in procs]
    got = q.get(timeout=120)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    A = O.synth_matrix(O.MAT_UNIFORM32, 9, m, k)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(9), k, n)
    assert got == O.matmul_f32(A, B).tobytes()


def _mm_gpu_worker(rank, world, port, m, k, n, prec, q):
    sys.path.insert(0, str(ROOT))
    from paper_1505_05655_b200 import device as D
    from paper_1505_05655_b200.shard import ShardedMatmul
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, nr = band(m, world, rank)
    k0, nk = band(k, world, rank)
    a = D.synth_matrix(1, 21, m, k, r0, nr)
    b = D.synth_matrix(1, 22, k, n, k0, nk)

    def mm(A, B):
        C = torch.empty(A.shape[0], n, device="cuda")
        D.matmul(prec, A, B, C, D.matmul_workspace(prec, A.shape[0], n, k))
        return C

    c = ShardedMatmul(dist, mm).run(a, b, k, n, world)
    full = gather_bands(dist, c.cpu(), [nr_ for _, nr_ in bands(m, world)], n)
    if rank == 0:
        q.put(full.numpy().tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [0, 2])  # f32 SIMT, bf16 tcgen05
@pytest.mark.parametrize("world,m,k,n", [(2, 1024, 768, 512), (3, 1000, 777, 520)])
def test_sharded_matmul_device_path_bitwise_invariant(gpu, prec, world, m, k, n):
    """The one-process-per-GPU MATMUL path with the sm_100a kernels: world
    2 / 3 processes on cuda:0 (gloo for the plumbing), block rows of A / C,
    B replicated from per-rank k-slices, C gathered -- bitwise equal to the
    single-device product (acceptance.cpp:278-315's invariance, carried to
    ranks)."""
    from paper_1505_05655_b200 import device as D
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mm_gpu_worker, args=(r, world, port, m, k, n, prec, q))
             for r in range(world)]
    [p.start() for p in procs]
    got = q.get(timeout=240)
    [p.join(timeout=120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    A = D.synth_matrix(1, 21, m, k)
    B = D.synth_matrix(1, 22, k, n)
    C = torch.empty(m, n, device="cuda")
    D.matmul(prec, A, B, C, D.matmul_workspace(prec, m, n, k))
    assert got == C.cpu().numpy().tobytes()
