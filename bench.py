#!/usr/bin/env python3
"""bench.py -- LUT-correction Gpixel/s (+ matmul TFLOP/s) on B200, next to the
host-CPU reference path.

Primary line (BASELINE.json metric): LUT image correction (LUT_GEN equalize +
LUT_APPLY, i.e. LUT_CORRECT) of the config-C3 scene, 32768 x 32768 u16
(ramp12 synthetic), row-band sharded over N GPUs: each rank histograms its
band, the 65536-bin histograms are summed (the one exchange step the
equalize LUT needs: inside the kernel over peer memory by default, NCCL as
the fallback), every rank builds the identical LUT and applies it to its
band.  One step = one full LUT_CORRECT of the scene.  Riding along in the
same JSON line: `stretch` (C3, mode=stretch), `demosaic` (§8f row 1),
`matmul` (C4 bf16 32768^3 + its tf32 variant, C2 f32 4096^3), `e2e`, `c5`
(64 chained requests through the server, with a phase breakdown), `c1`
(one request over TCP and through the C ABI) and the CPU baselines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
  python bench.py --gpc-bench --task T [--dims ...] [--workers-list ...]

Timing: CUDA events on the stream the kernels are launched on, barrier +
synchronize on both sides of the K timed steps, max over ranks.  Inputs are
device-resident and larger than L2 (2 GiB / N per rank) -- no flush needed.
`e2e` runs the same LUT_CORRECT through the C ABI (gpcx_lut_host) with
pinned HOST buffers: H2D + kernels + D2H inside the timed region, on rank 0
with all N GPUs bound in-process (the server's architecture).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LUT-correction Gpixel/s + matmul TFLOP/s at 1/2/4/8 B200 vs host CPU ref"
ROWS = COLS = 32768
SEED = 0x5EED
MM = 4096  # config C2


def splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


SEED_B = splitmix64(SEED)  # seed of matrix B (same derivation as the library's tests)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


class Clocks:
    """NVML sampler (the data nvidia-smi's clocks line reports) polling every
    2 ms during the timed region -- the LUT step is ~1 ms, far below
    nvidia-smi's sampling period -- plus one sample at entry and exit."""

    REASONS = {  # nvmlClocksEventReasons bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
    }

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nv = None

    def _sample(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((sm, rs))

    def _loop(self):
        while not self._stop.wait(0.002):
            self._sample()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._sample()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception:  # no NVML: report no samples rather than guess
            self._nv = None
        return self

    def __exit__(self, *exc):
        if self._nv is not None:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self) -> dict:
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "NVML, 2 ms polling"}


# ------------------------------------------------------------------ dist ---

class Dist:
    def __init__(self, want: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if want != self.world and self.world != 1:
            raise SystemExit(f"--gpus {want} but WORLD_SIZE={self.world}")
        if want > 1 and self.world == 1 and os.environ.get("GPCX_BENCH_SINGLE_PROCESS") != "1":
            # one process would time only its own band while `value` counts
            # the whole scene -- N > 1 is one process per GPU
            raise SystemExit(f"--gpus {want} needs one process per GPU: "
                             f"torchrun --nproc-per-node {want} bench.py --gpus {want}")
        self.n = want if self.world == 1 else self.world
        self.pg = None

    # GPCX_BENCH_ONE_GPU=1 (testing only): every rank on cuda:0 over gloo, so
    # the N>1 code path can be exercised on a single-GPU box.
    one_gpu = os.environ.get("GPCX_BENCH_ONE_GPU") == "1"

    @property
    def gpu(self) -> int:
        return 0 if self.one_gpu else self.local

    def init(self, backend: str):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            if backend == "nccl" and not self.one_gpu:
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                torch.cuda.set_device(self.gpu)
                dist.init_process_group("gloo")
            self.pg = dist

    def all_reduce_(self, t):
        """In-place sum over ranks (NCCL on the device; via host for gloo)."""
        if self.pg is None:
            return
        if self.pg.get_backend() == "nccl":
            self.pg.all_reduce(t)
        else:
            h = t.cpu()
            self.pg.all_reduce(h)
            t.copy_(h)

    def sum_u64(self, x: int) -> int:
        """Sum of a Python int over ranks, mod 2^64 (band digests)."""
        if self.pg is None:
            return x
        xs = [None] * self.n
        self.pg.all_gather_object(xs, x)
        return sum(xs) & (2 ** 64 - 1)

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if self.pg.get_backend() == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


def bound_devices(n: int) -> list[int]:
    """Devices the in-process legs bind: 0..n-1 (device 0 n times in the
    GPCX_BENCH_ONE_GPU test mode -- the planner's multi-band path)."""
    return [0] * n if Dist.one_gpu else list(range(n))


def band(rows: int, n: int, r: int) -> tuple[int, int]:
    per = (rows + n - 1) // n
    r0 = min(rows, r * per)
    return r0, min(per, rows - r0)


# ------------------------------------------------------------- B200 legs ---

def exchange_mode(d: Dist) -> str:
    """N>1 histogram exchange: "peer" (fused into the kernel over NVLink peer
    memory, gpcx_lut_peer_*) unless GPCX_LUT_EXCHANGE=nccl; the single-GPU
    test mode defaults to the NCCL/gloo path (its ranks share one GPU and
    would meet only through time-slicing)."""
    want = os.environ.get("GPCX_LUT_EXCHANGE", "")
    if want in ("peer", "nccl"):
        return want
    return "nccl" if Dist.one_gpu else "peer"


def open_peer_exchange(d: Dist, make_peer, dev):
    """Create this rank's exchange block, all-gather the IPC handles and
    connect -- or, if ANY rank fails (no P2P path, allocation failure),
    return None on every rank so all of them use the NCCL exchange."""
    import torch
    peer = mine = None
    try:
        peer = make_peer()
        mine = peer.handle()
    except Exception as e:
        print(f"rank {d.rank}: peer exchange unavailable ({e}); using NCCL", file=sys.stderr)
    handles = [None] * d.n
    d.pg.all_gather_object(handles, mine)  # every rank takes part, even after a failure
    ok = int(all(h is not None for h in handles))
    if ok:
        try:
            peer.connect(handles)
        except Exception as e:
            print(f"rank {d.rank}: peer exchange unavailable ({e}); using NCCL", file=sys.stderr)
            ok = 0
    flag = torch.tensor([ok], dtype=torch.int32,
                        device=dev if d.pg.get_backend() == "nccl" else "cpu")
    d.pg.all_reduce(flag, op=d.pg.ReduceOp.MIN)
    if int(flag.item()) == 0:
        if peer is not None:
            peer.close()
        return None
    return peer


def lut_device_leg(d: Dist, steps: int, warmup: int, mode: int, gather: bool = True) -> dict:
    import torch
    from paper_1505_05655_b200 import device as D
    dev = torch.device("cuda", d.gpu)
    torch.cuda.set_device(dev)
    r0, nr = band(ROWS, d.n, d.rank)
    n = nr * COLS
    img = D.synth_image(0, SEED, ROWS, COLS, r0, nr)
    out = torch.empty_like(img)
    hist = torch.zeros(65536, dtype=torch.int32, device=dev)
    lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
    stream = torch.cuda.current_stream()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev = {k: [] for k in ("h0", "h1", "a0", "a1")}
    peer = None
    if d.pg is not None and exchange_mode(d) == "peer":
        # histogram exchange fused into the kernel over peer memory: IPC
        # handles of every rank's exchange block, all-gathered once
        peer = open_peer_exchange(d, lambda: D.LutPeer(d.rank, d.n), dev)

    def step(record: bool):
        if record:
            ev["h0"].append(E()); ev["h0"][-1].record(stream)
        if d.pg is None:  # one GPU: ONE cooperative launch (histogram -> LUT -> apply)
            D.lut_correct(img, out, mode, lut, stats, ws, stream)
            if record:
                ev["h1"].append(E()); ev["h1"][-1].record(stream)
            return
        if peer is not None:  # N GPUs, still ONE launch per rank per step
            peer.correct(img, out, mode, lut, stats, ws, stream)
            if record:
                ev["h1"].append(E()); ev["h1"][-1].record(stream)
            return
        # N GPUs: local histogram (fused_kernel, count stage), NCCL all-reduce
        # of the 256 KiB histogram, then LUT + apply of the band (one launch)
        D.lut_hist(img, hist, ws, stream)
        if record:
            ev["a0"].append(E()); ev["a0"][-1].record(stream)
        d.all_reduce_(hist)
        if record:
            ev["a1"].append(E()); ev["a1"][-1].record(stream)
        D.lut_correct_from_hist(hist, mode, img, out, lut, stats, ws, stream)
        if record:
            ev["h1"].append(E()); ev["h1"][-1].record(stream)

    for _ in range(warmup):
        step(False)
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    t0, t1 = E(), E()
    with Clocks(d.gpu) as clk:
        t0.record(stream)
        for _ in range(steps):
            step(True)
        t1.record(stream)
        torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    hist_ms = sum(a.elapsed_time(b) for a, b in zip(ev["h0"], ev["h1"])) / steps
    # N>1: time spent in the histogram all-reduce (between the two launches)
    exch_ms = (sum(a.elapsed_time(b) for a, b in zip(ev["a0"], ev["a1"])) / steps
               if ev["a0"] else None)
    # correctness guard on the measured buffers (device digest vs nothing
    # here; the oracle check of this exact band runs in the cpu leg).
    # parity of the timed output: the band's position-keyed digest (additive
    # over bands), summed over ranks and compared with the oracle's by rank 0
    dig = int(D.digest_u16(out, r0 * COLS).item()) & (2 ** 64 - 1)
    dig = d.sum_u64(dig)
    st = D.read_stats(stats)
    gather_ms = gather_leg(d, out) if d.pg is not None and gather else None
    if peer is not None:
        d.barrier()  # no rank unmaps its exchange block while a peer may still read it
        torch.cuda.synchronize()
        peer.close()
    return {"ms": ms, "hist_ms": hist_ms, "exch_ms": exch_ms, "band_px": n, "digest": dig,
            "stats": st, "clocks": clk.summary(), "gather_ms": gather_ms,
            "exchange": None if d.pg is None else ("peer" if peer is not None else "nccl")}


def gather_leg(d: Dist, out, reps: int = 3) -> float:
    """N>1: the final gather of the corrected bands to rank 0 (NCCL over
    NVLink; paper_1505_05655_b200.shard.gather_bands), timed on its own --
    SURVEY.md §8e: sharded-compute scaling is reported separately from the
    gather.  Max over ranks of the mean of `reps` gathers."""
    import torch
    from paper_1505_05655_b200.shard import gather_bands
    rows_per = [band(ROWS, d.n, r)[1] for r in range(d.n)]
    nccl = d.pg.get_backend() == "nccl"
    src = out if nccl else out.cpu()
    gather_bands(d.pg, src, rows_per, COLS)  # warm-up (communicator buffers)
    d.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        full = gather_bands(d.pg, src, rows_per, COLS)
        torch.cuda.synchronize()
        del full
    ms = (time.perf_counter() - t) * 1e3 / reps
    d.barrier()
    return ms


def lut_e2e_leg(n_gpus: int, steps: int, warmup: int, mode: int, inflight: int = 1) -> dict:
    """Rank 0, all N GPUs bound in-process: gpcx_lut_host with pinned host
    buffers (H2D + kernels + D2H per step).  `inflight` requests are issued
    concurrently from that many host threads (a server with several requests
    queued): one request's H2D then overlaps another's D2H on the
    full-duplex PCIe link.  value = scenes corrected per second x pixels."""
    import ctypes as C
    import threading as th
    import torch
    import paper_1505_05655_b200 as G
    from paper_1505_05655_b200 import device as D
    G.init(bound_devices(n_gpus))
    n = ROWS * COLS
    bufs = [(G.lib.gpcx_pinned_alloc(n * 2), G.lib.gpcx_pinned_alloc(n * 2)) for _ in range(inflight)]
    try:
        scene = D.synth_image(0, SEED, ROWS, COLS).cpu().numpy().view(np.uint16)
        for p_in, _ in bufs:
            np.ctypeslib.as_array((C.c_uint16 * n).from_address(p_in))[:] = scene
        del scene
        torch.cuda.empty_cache()

        def one(p_in, p_out):
            st = G.LutStats()
            G.check(G.lib.gpcx_lut_host(2, mode, ROWS, COLS, C.c_void_p(p_in), None,
                                        C.c_void_p(p_out), None, C.byref(st)))

        def worker(k, p_in, p_out, count):
            for _ in range(count):
                one(p_in, p_out)

        for _ in range(warmup):  # at full concurrency: one request slot per in-flight request
            ws = [th.Thread(target=worker, args=(k, *bufs[k], 1)) for k in range(inflight)]
            [x.start() for x in ws]
            [x.join() for x in ws]
        per = max(1, steps // inflight)
        t = time.perf_counter()
        ts = [th.Thread(target=worker, args=(k, *bufs[k], per)) for k in range(inflight)]
        [x.start() for x in ts]
        [x.join() for x in ts]
        wall = time.perf_counter() - t
    finally:
        for p_in, p_out in bufs:
            G.lib.gpcx_pinned_free(p_in)
            G.lib.gpcx_pinned_free(p_out)
        G.init([0])
    done = per * inflight
    return {"value": n * done / wall / 1e9, "ms_per_step": 1e3 * wall / done,
            "h2d_bytes_per_step": n * 2, "d2h_bytes_per_step": n * 2, "inflight": inflight}


# config C4 (GPCX_BENCH_MM4 shrinks it for the GPCX_BENCH_ONE_GPU dry run
# only: 8 ranks replicating a 4 GiB B over gloo through host memory)
MM4 = int(os.environ.get("GPCX_BENCH_MM4", "32768")) if os.environ.get("GPCX_BENCH_ONE_GPU") == "1" \
    else 32768
C4_SAMPLE_ROWS, C4_SAMPLE_COLS = 128, 512  # CPU baseline / parity sample of C


def matmul_c4_leg(d: Dist, steps: int, warmup: int, prec: int = 2) -> dict:
    """Config C4: 32768^3 MATMUL on the tcgen05 path, block rows of A / C per
    rank.  B is REPLICATED every step: rank r holds only its
    k-slice of B's rows (generated in place -- what its own PCIe link would
    stage) and the slices are all-gathered (NCCL over NVLink;
    shard.replicate_rows) into a double-buffered full B on a side stream, so
    step s+1's replication runs under step s's GEMM.  One step = replicate
    B + the rank's block-row product including the f32 -> bf16 operand
    preparation.  `ms` is that pipelined step; `compute_ms` the product
    alone; `replicate_ms` one replication timed by itself (N>1)."""
    import torch
    from paper_1505_05655_b200 import device as D
    from paper_1505_05655_b200.shard import replicate_rows
    r0, nr = band(MM4, d.n, d.rank)
    k0, nk = band(MM4, d.n, d.rank)
    kslices = [band(MM4, d.n, r)[1] for r in range(d.n)]
    A = D.synth_matrix(1, SEED, MM4, MM4, r0, nr)
    Cm = torch.empty(nr, MM4, device="cuda")
    ws = D.matmul_workspace(prec, nr, MM4, MM4)
    stream = torch.cuda.current_stream()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    sharded = d.pg is not None
    if sharded:
        own = D.synth_matrix(1, SEED_B, MM4, MM4, k0, nk)
        bufs = [torch.empty(MM4, MM4, device="cuda") for _ in range(2)]
        comm = torch.cuda.Stream()
    else:  # one rank owns all of B: nothing to replicate
        bufs = [D.synth_matrix(1, SEED_B, MM4, MM4)]

    def replicate(buf, after=None):
        with torch.cuda.stream(comm):
            if after is not None:
                comm.wait_event(after)
            replicate_rows(d.pg, own, kslices, MM4, out=buf)
            ev = torch.cuda.Event()
            ev.record(comm)
        return ev

    def run(n_steps: int, record: bool):
        """n_steps pipelined steps; returns per-step compute events."""
        done = [None, None]
        ready = replicate(bufs[0]) if sharded else None
        spans = []
        for s in range(n_steps):
            b = bufs[s % len(bufs)]
            if ready is not None:
                stream.wait_event(ready)
            if sharded and s + 1 < n_steps:  # next step's B, under this GEMM
                ready = replicate(bufs[(s + 1) % 2], after=done[(s + 1) % 2])
            a0 = E() if record else None
            if record:
                a0.record(stream)
            D.matmul(prec, A, b, Cm, ws, stream)
            ev = torch.cuda.Event(enable_timing=record)
            ev.record(stream)
            done[s % 2] = ev
            if record:
                spans.append((a0, ev))
        return spans

    run(warmup, False)
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    t0, t1 = E(), E()
    with Clocks(d.gpu) as clk:
        t0.record(stream)
        spans = run(steps, True)
        t1.record(stream)
        torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    compute_ms = sum(a.elapsed_time(b) for a, b in spans) / steps
    rep_ms = None
    if sharded:  # one replication by itself (not under a GEMM)
        d.barrier()
        torch.cuda.synchronize()
        a, b = E(), E()
        a.record(comm)
        with torch.cuda.stream(comm):
            replicate_rows(d.pg, own, kslices, MM4, out=bufs[0])
        b.record(comm)
        torch.cuda.synchronize()
        rep_ms = a.elapsed_time(b)
    B = bufs[(steps - 1) % len(bufs)]
    # rank 0 keeps a 128 x 512 corner of the product (and its operands) for
    # the CPU baseline and a sampled parity check against the f64 oracle
    sample = None
    if d.rank == 0:
        sample = {"A": A[:C4_SAMPLE_ROWS].cpu().numpy(),
                  "B": B[:, :C4_SAMPLE_COLS].contiguous().cpu().numpy(),
                  "C": Cm[:C4_SAMPLE_ROWS, :C4_SAMPLE_COLS].cpu().numpy(), "prec": prec}
    del A, B, ws, bufs
    if sharded:
        del own
    gather_ms = None
    if d.pg is not None:  # the C bands to rank 0, timed apart from the compute
        from paper_1505_05655_b200.shard import gather_bands
        rows_per = [band(MM4, d.n, r)[1] for r in range(d.n)]
        src = Cm if d.pg.get_backend() == "nccl" else Cm.cpu()
        gather_bands(d.pg, src, rows_per, MM4)
        d.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        full = gather_bands(d.pg, src, rows_per, MM4)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - t) * 1e3
        del full, src
        d.barrier()
    del Cm
    torch.cuda.empty_cache()
    return {"ms": ms, "compute_ms": compute_ms, "replicate_ms": rep_ms, "rows": nr,
            "clocks": clk.summary(), "gather_ms": gather_ms, "sample": sample}


def matmul_device_leg(steps: int, warmup: int) -> dict:
    """Config C2: FP32 4096^3 on the SIMT reference-precision kernel; L2 is
    flushed (256 MiB write) between steps, outside the GEMM events."""
    import torch
    from paper_1505_05655_b200 import device as D
    A = D.synth_matrix(1, SEED, MM, MM)
    B = D.synth_matrix(1, SEED_B, MM, MM)
    Cm = torch.empty(MM, MM, device="cuda")
    ws = D.matmul_workspace(0, MM, MM, MM)  # A^T for the SIMT kernel
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    times = []
    with Clocks(torch.cuda.current_device()) as clk:
        for i in range(warmup + steps):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            D.matmul(0, A, B, Cm, ws, stream)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= warmup:
                times.append(a.elapsed_time(b))
    ms = sum(times) / len(times)
    flops = 2.0 * MM ** 3
    return {"ms": ms, "tflops": flops / ms / 1e9, "C": Cm, "clocks": clk.summary()}


def matmul_e2e_leg(steps: int) -> dict:
    import ctypes as C
    import paper_1505_05655_b200 as G
    from paper_1505_05655_b200 import device as D
    A = D.synth_matrix(1, SEED, MM, MM).cpu().numpy()
    B = D.synth_matrix(1, SEED_B, MM, MM).cpu().numpy()
    nb = MM * MM * 4
    pa, pb, pc = (G.lib.gpcx_pinned_alloc(nb) for _ in range(3))
    try:
        np.ctypeslib.as_array((C.c_float * (MM * MM)).from_address(pa))[:] = A.ravel()
        np.ctypeslib.as_array((C.c_float * (MM * MM)).from_address(pb))[:] = B.ravel()
        times = []
        for i in range(steps + 1):
            t = time.perf_counter()
            G.check(G.lib.gpcx_matmul_host(0, MM, MM, MM, C.c_void_p(pa), C.c_void_p(pb), C.c_void_p(pc)))
            if i:
                times.append(time.perf_counter() - t)
    finally:
        for p in (pa, pb, pc):
            G.lib.gpcx_pinned_free(p)
    s = sum(times) / len(times)
    return {"value": 2.0 * MM ** 3 / s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 2 * nb,
            "d2h_bytes_per_step": nb}


# ------------------------------------------------------------ demosaic ---

DM = 16384  # BAYER_* device leg: 16384^2 u16 mosaic (512 MiB in, 1.5 GiB out > L2)


def demosaic_leg(steps: int, warmup: int) -> dict:
    """BAYER_BILINEAR / BAYER_GRADIENT (RGGB) on a
    16384^2 uniform16 mosaic, device-resident, CUDA events on the launch
    stream; 8 B/px algorithmic (2 in + 6 out), inputs + outputs > L2."""
    import torch
    from paper_1505_05655_b200 import device as D
    img = D.synth_image(1, SEED, DM, DM)
    out = torch.empty(3 * DM * DM, dtype=torch.int16, device="cuda")
    stream = torch.cuda.current_stream()
    res = {}
    for name, grad in (("bilinear", False), ("gradient", True)):
        times = []
        with Clocks(torch.cuda.current_device()) as clk:
            for i in range(warmup + steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                D.demosaic(grad, 0, img, DM, DM, out, stream)
                b.record(stream)
                torch.cuda.synchronize()
                if i >= warmup:
                    times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        res[name] = {"ms": ms, "clocks": clk.summary()}
    del img, out
    torch.cuda.empty_cache()
    return res


def demosaic_task_leg(reps: int = 5) -> dict:
    """BAYER_BILINEAR through the task-level C ABI (gpcx_run) with pinned
    host buffers at 8192^2 (128 MiB request, 384 MiB response: under the
    1 GiB wire cap): H2D + kernel + D2H per request."""
    import ctypes as C
    import paper_1505_05655_b200 as G
    n = 8192
    nin, nout = 2 * n * n, 6 * n * n
    pin, pout = G.lib.gpcx_pinned_alloc(nin), G.lib.gpcx_pinned_alloc(nout)
    try:
        img = np.ctypeslib.as_array((C.c_uint16 * (n * n)).from_address(pin))
        img[:] = np.random.default_rng(SEED).integers(0, 1 << 16, n * n, dtype=np.uint16)
        out = np.ctypeslib.as_array((C.c_uint8 * nout).from_address(pout))
        times = []
        for i in range(reps + 1):
            t = time.perf_counter()
            G.run("BAYER_BILINEAR", f"rows={n},cols={n}", img, out)
            if i:
                times.append(time.perf_counter() - t)
    finally:
        G.lib.gpcx_pinned_free(pin)
        G.lib.gpcx_pinned_free(pout)
    s = statistics.median(times)
    return {"value": n * n / s / 1e9, "unit": "Gpixel/s", "ms": round(1e3 * s, 2),
            "h2d_bytes_per_step": nin, "d2h_bytes_per_step": nout,
            "path": f"gpcx_run BAYER_BILINEAR rows={n},cols={n}, pinned host buffers, median of {reps}"}


# ------------------------------------------------------------------ C5 ---

# Chain sizes: the C1 image (4096^2 u16) and the C2 product (4096^3), so each
# chain is LUT_GEN + LUT_APPLY of C1 and a MATMUL of the corrected image
# (as f32 in [0,1]) with B -- 290 MB over TCP and 137 GFLOP per chain.
C5_IMG = 4096
C5_MM = 4096
C5_REQUESTS = 64
C5_CPU_SAMPLE = 16  # chains timed on the reference CPU server (bounded sample)


def c5_inputs(count: int = C5_REQUESTS) -> tuple[list[bytes], bytes]:
    from paper_1505_05655_b200 import device as D
    imgs = [D.synth_image(0, SEED + i, C5_IMG, C5_IMG).cpu().numpy().view(np.uint16).tobytes()
            for i in range(count)]
    B = D.synth_matrix(1, SEED_B, C5_MM, C5_MM).cpu().numpy().tobytes()
    return imgs, B


def c5_chain(port: int, img: bytes, B: bytes, prec: str) -> int:
    """LUT_GEN -> LUT_APPLY (image correction) -> MATMUL on the corrected
    image's top-left block; returns the bytes moved over TCP.  The client is
    libgpcx's native one (gpcx_client_submit, the reference client's
    protocol) so the load generator's socket I/O runs off the GIL."""
    from paper_1505_05655_b200.client import submit_native as submit
    dims = f"rows={C5_IMG},cols={C5_IMG}"
    lut = np.empty(131072, dtype=np.uint8)
    r1 = submit("127.0.0.1", port, "LUT_GEN", dims, [img], output_name="lut.bin", out=lut)
    assert r1.ok, r1.status
    corr = np.empty(C5_IMG * C5_IMG, dtype=np.uint16)
    r2 = submit("127.0.0.1", port, "LUT_APPLY", dims, [lut, img], output_name="img.raw",
                out=corr.view(np.uint8))
    assert r2.ok, r2.status
    A = corr.reshape(C5_IMG, C5_IMG)[:C5_MM, :C5_MM].astype(np.float32)
    A *= np.float32(1.0 / 65535.0)
    cm = np.empty(C5_MM * C5_MM, dtype=np.float32)
    r3 = submit("127.0.0.1", port, "MATMUL", f"m={C5_MM},k={C5_MM},n={C5_MM},prec={prec}", [A, B],
                output_name="c.f32", out=cm.view(np.uint8))
    assert r3.ok, r3.status
    return (len(img) * 2 + len(r1.payload) + A.nbytes + len(B) + len(r1.payload) + len(r2.payload)
            + len(r3.payload) + 6 * 260)


def c5_run(port: int, imgs, B, prec: str, clients: int = C5_REQUESTS) -> dict:
    """All chains submitted at once by `clients` client threads (queued at
    the server, which runs max_tasks of them concurrently)."""
    import concurrent.futures as cf
    t = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=clients) as ex:
        moved = sum(ex.map(lambda im: c5_chain(port, im, B, prec), imgs))
    s = time.perf_counter() - t
    return {"chains": len(imgs), "chains_per_s": len(imgs) / s, "requests_per_s": 3 * len(imgs) / s,
            "seconds": s, "tcp_bytes": moved}


def c5_leg(n_gpus: int) -> dict:
    """Config C5: 64 queued client requests, each the chain LUT_GEN ->
    LUT_APPLY -> MATMUL, against the B200 task server (N GPUs bound in one
    server process, requests round-robined over them)."""
    import paper_1505_05655_b200 as G
    imgs, B = c5_inputs()
    G.init(bound_devices(n_gpus))
    try:
        with G.Server(max_tasks=0) as srv:
            # warm-up at the full concurrency: the first pass grows the
            # server's request slots (device buffers) and pinned pools to 64
            # requests in flight -- 3-6x slower than steady state
            # (tools/c5_probe.py), and not what a running server pays
            c5_run(srv.port, imgs, B, "bf16")
            st0 = srv.stats()
            res = c5_run(srv.port, imgs, B, "bf16")
            st1 = srv.stats()
    finally:
        G.init([0])
    nreq = max(1, st1["requests"] - st0["requests"])
    res["phases_ms_per_request"] = {
        k: round((st1[k] - st0[k]) / nreq, 3) for k in ("recv_ms", "task_ms", "send_ms")}
    res["phases_note"] = ("server-side, averaged over the timed pass's requests: payload "
                          "received (TCP, H2D chunks overlapped) | task work after the last "
                          "payload byte (kernels, D2H) | response written (TCP)")
    res.update({"workload": f"C5: {C5_REQUESTS} concurrent clients x (LUT_GEN -> LUT_APPLY -> "
                            f"MATMUL prec=bf16), {C5_IMG}^2 u16 images, {C5_MM}^3 matmul",
                "server": "gpcx B200 server (max_tasks = 2 x hw threads), loopback TCP, "
                          "native client (gpcx_client_submit) driven from 64 threads"})
    return res


def c1_run(port: int, img: bytes, reps: int, warmup: int = 2) -> dict:
    """Config C1: ONE client request at a time -- LUT_CORRECT of a 4096^2
    u16 image over loopback TCP (260-byte header + 32 MiB up, 32 MiB down),
    latency per request; the native client (gpcx_client_submit)."""
    from paper_1505_05655_b200.client import submit_native as submit
    out = np.empty(C5_IMG * C5_IMG, dtype=np.uint16)
    dims = f"rows={C5_IMG},cols={C5_IMG},mode=equalize"
    ts = []
    for i in range(warmup + reps):
        t = time.perf_counter()
        r = submit("127.0.0.1", port, "LUT_CORRECT", dims, [img], output_name="c1.raw",
                   out=out.view(np.uint8))
        assert r.ok, r.status
        if i >= warmup:
            ts.append(time.perf_counter() - t)
    ms = statistics.median(ts) * 1e3
    return {"ms_per_request": round(ms, 3), "Gpixel/s": round(C5_IMG * C5_IMG / ms / 1e6, 3),
            "requests": reps, "digest": int(np.frombuffer(out.tobytes(), dtype=np.uint64).sum(
                dtype=np.uint64))}


def served_leg(n_gpus: int, reps: int = 5, matmul: bool = True) -> dict:
    """The over-cap configs through the SERVED path (SURVEY.md §8d option ii):
    header-only requests (synth=..., no payload) from the native client over
    loopback TCP to the B200 server with all N GPUs bound.  C3: LUT_CORRECT
    of the 32768^2 ramp12 scene generated on the GPUs, answered with the
    corrected image's digest (checked against the oracle by the caller);
    C4: MATMUL 32768^3 bf16, answered with 4096 seeded samples of C.  Per
    request: generation (2 B/px / 8 B per matrix element written) + the task
    + an 8-byte / 48 KiB response; median of `reps` after one warm-up."""
    import struct
    import paper_1505_05655_b200 as G
    from paper_1505_05655_b200.client import submit_native as submit
    G.init(bound_devices(n_gpus))
    res = {}
    try:
        with G.Server(max_tasks=0) as srv:
            params = f"rows={ROWS},cols={COLS},mode=equalize,synth=ramp12,seed={SEED}"
            ts, digest = [], None
            for i in range(reps + 1):
                t = time.perf_counter()
                r = submit("127.0.0.1", srv.port, "LUT_CORRECT", params, [], resp_cap=8,
                           output_name="c3.digest")
                assert r.ok, r.status
                if i:
                    ts.append(time.perf_counter() - t)
                digest = struct.unpack("<Q", bytes(r.payload))[0]
            ms = statistics.median(ts) * 1e3
            res["c3"] = {"request": f"LUT_CORRECT {params} (no payload)", "ms_per_request": round(ms, 3),
                         "value": round(ROWS * COLS / ms / 1e6, 2), "unit": "Gpixel/s",
                         "includes": "scene generation on the GPUs (2 B/px written) + LUT_CORRECT + digest",
                         "digest": digest}
            if matmul:
                mparams = f"m={MM4},k={MM4},n={MM4},prec=bf16,synth=uniform32,seed={SEED}"
                ts = []
                for i in range(3):
                    t = time.perf_counter()
                    r = submit("127.0.0.1", srv.port, "MATMUL", mparams, [], resp_cap=4096 * 12,
                               output_name="c4.samples")
                    assert r.ok, r.status
                    if i:
                        ts.append(time.perf_counter() - t)
                ms = statistics.median(ts) * 1e3
                res["c4"] = {"request": f"MATMUL {mparams} (no payload)", "ms_per_request": round(ms, 3),
                             "value": round(2.0 * MM4 ** 3 / ms / 1e9, 1), "unit": "TFLOP/s",
                             "includes": "A / B generation on the GPUs + operand prep + GEMM + 4096 samples"}
    finally:
        G.init([0])
    return res


def c1_leg(n_gpus: int) -> dict:
    import paper_1505_05655_b200 as G
    imgs, _ = c5_inputs(count=1)
    G.init(bound_devices(n_gpus))
    try:
        with G.Server(max_tasks=0) as srv:
            res = c1_run(srv.port, imgs[0], reps=20)
    finally:
        G.init([0])
    res["workload"] = ("C1: one LUT_CORRECT request (4096^2 u16, equalize) at a time through the "
                       "B200 server, loopback TCP, median latency")
    res["direct"] = c1_direct(imgs[0])
    return res


def c1_direct(img: bytes, reps: int = 20) -> dict:
    """The same C1 request through the task-level C ABI (gpcx_run) from
    pinned host buffers -- the server's work without the sockets: 32 MiB
    H2D, the fused LUT kernel, 32 MiB D2H."""
    import ctypes as C
    import paper_1505_05655_b200 as G
    n = C5_IMG * C5_IMG
    pin, pout = G.lib.gpcx_pinned_alloc(2 * n), G.lib.gpcx_pinned_alloc(2 * n)
    try:
        src = np.ctypeslib.as_array((C.c_uint16 * n).from_address(pin))
        src[:] = np.frombuffer(img, dtype=np.uint16)
        dst = np.ctypeslib.as_array((C.c_uint8 * (2 * n)).from_address(pout))
        ts = []
        for i in range(reps + 2):
            t = time.perf_counter()
            G.run("LUT_CORRECT", f"rows={C5_IMG},cols={C5_IMG},mode=equalize", src, dst)
            if i >= 2:
                ts.append(time.perf_counter() - t)
    finally:
        G.lib.gpcx_pinned_free(pin)
        G.lib.gpcx_pinned_free(pout)
    ms = statistics.median(ts) * 1e3
    return {"ms_per_request": round(ms, 3), "Gpixel/s": round(n / ms / 1e6, 3),
            "h2d_bytes": 2 * n, "d2h_bytes": 2 * n,
            "path": "gpcx_run LUT_CORRECT, pinned host buffers, median of 20"}


# -------------------------------------------------------------- CPU legs ---

def cpu_c5() -> dict:
    """C5 against the reference server (the reference's own TCP / dispatch
    code, proj/src/server.cpp) serving the CPU-restated tasks."""
    from oracle import oracle as O
    imgs, B = c5_inputs()
    with O.RefServer(max_tasks=0) as rs:
        c5_run(rs.port, imgs[:4], B, "bf16", 4)  # warm-up (no pools to grow: a short one)
        res = c5_run(rs.port, imgs[:C5_CPU_SAMPLE], B, "bf16", C5_CPU_SAMPLE)
    res.update({"kind": "port", "cores": O.max_threads(),
                "sample": f"the first {C5_CPU_SAMPLE} chains of the same corpus, {C5_CPU_SAMPLE} concurrent "
                          "clients, through the reference server "
                          "(oracle/_ref: reference server + restated CPU kernels)"})
    return res

def cpu_c1() -> dict:
    """C1 against the reference server (its TCP / dispatch code, the restated
    LUT_CORRECT on all host cores)."""
    from oracle import oracle as O
    imgs, _ = c5_inputs(count=1)
    with O.RefServer(max_tasks=0) as rs:
        res = c1_run(rs.port, imgs[0], reps=5, warmup=1)
    res.update({"kind": "port", "cores": O.max_threads(),
                "sample": "5 sequential requests after 1 warm-up, same image and client"})
    px = np.frombuffer(imgs[0], dtype=np.uint16)
    ts = []
    for i in range(6):
        t = time.perf_counter()
        O.lut_correct(px, O.LUT_EQUALIZE)
        if i:
            ts.append(time.perf_counter() - t)
    ms = statistics.median(ts) * 1e3
    res["direct"] = {"ms_per_request": round(ms, 3), "Gpixel/s": round(px.size / ms / 1e6, 3),
                     "path": "oracle/gpcx_oracle.c LUT_CORRECT in process, every host thread, "
                             "median of 5"}
    return res


def c3_config(n: int) -> dict:
    """The C3 workload as both arms name it (`same_config`)."""
    return {"workload": "C3: LUT_CORRECT equalize, 32768x32768 u16 scene, row bands",
            "rows": ROWS, "cols": COLS, "mode": "equalize", "image": "ramp12",
            "parallelism": f"row-band x{n}", "l2": "inputs larger than L2 (2 GiB scene)"}


def cpu_lut_full(modes=(0, 1), reps: int = 3, threads: int = 0) -> dict:
    """The restated oracle (kind "port"; the reference has no LUT code) on
    the WHOLE C3 scene with every host thread: per mode the median
    LUT_CORRECT time over `reps` runs, the output's position-keyed digest
    and the stats -- the CPU baseline and the parity reference of the timed
    GPU output at once."""
    from oracle import oracle as O
    threads = threads or O.max_threads()
    scene = O.synth_image(O.IMG_RAMP12, SEED, ROWS, COLS)
    res = {}
    for mode in modes:
        times = []
        for _ in range(reps):
            t = time.perf_counter()
            out, _, st = O.lut_correct(scene, mode, threads=threads)
            times.append(time.perf_counter() - t)
        res[mode] = {"s": statistics.median(times), "digest": O.digest_u16(out), "stats": st,
                     "reps": reps}
        del out
    res["cores"] = threads
    return res


def lut_parity(leg: dict, ref: dict) -> dict:
    """Timed GPU output vs the oracle on the same scene: bit-exact through
    the position-keyed u64 digest (sum over all 2^30 pixels) and the stats."""
    ok = leg["digest"] == ref["digest"] and leg["stats"] == ref["stats"]
    return {"ok": bool(ok), "digest": f"{leg['digest']:016x}", "oracle_digest": f"{ref['digest']:016x}",
            "stats": leg["stats"], "how": "sum_i splitmix64(i ^ out[i]) mod 2^64 over the whole "
                                          "timed output vs oracle/gpcx_oracle.c LUT_CORRECT of the scene"}


def cpu_lut(ref: dict, mode: int) -> dict:
    from oracle import oracle as O
    r = ref[mode]
    return {"value": ROWS * COLS / r["s"] / 1e9, "unit": "Gpixel/s", "cores": ref["cores"],
            "kind": "port",
            "sample": f"LUT_CORRECT {'equalize' if mode == 0 else 'stretch'} of the whole {ROWS}x{COLS} "
                      f"C3 scene (no sampling), median of {r['reps']}, oracle/gpcx_oracle.c with "
                      f"{ref['cores']} OpenMP threads",
            "host": O.host_cpu()}


def cpu_matmul(sample_rows: int = 64) -> dict:
    from oracle import oracle as O
    A = O.synth_matrix(O.MAT_UNIFORM32, SEED, MM, MM)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(SEED), MM, MM)
    rows = A[:sample_rows].copy()
    t = time.perf_counter()
    O.matmul_f32(rows, B)
    s = time.perf_counter() - t
    return {"value": 2.0 * sample_rows * MM * MM / s / 1e12, "unit": "TFLOP/s",
            "cores": O.max_threads(), "kind": "port",
            "sample": f"{sample_rows} rows of the C2 4096^3 FP32 product (f64 accumulate)"}


# ----------------------------------------------------------------- main ---

def cpu_matmul_c4(sample: dict) -> dict:
    """the C4 product is infeasible on the CPU (7e13 flop), so
    the oracle port times a 128 x 512 corner of it (full K = 32768, every
    host thread), and the same corner of the GPU's C is checked against the
    f64 oracle on bf16-rounded operands (tolerance 1e-5 * sum|a||b|)."""
    from oracle import oracle as O
    A, B, C = sample["A"], sample["B"], sample["C"]
    t = time.perf_counter()
    O.matmul_f32(A, B)
    s = time.perf_counter() - t
    prec = {2: O.PREC_BF16, 1: O.PREC_TF32}.get(sample["prec"], O.PREC_F32)
    Cref, ab = O.matmul_f64(O.round_matrix(prec, A), O.round_matrix(prec, B))
    err = np.abs(C.astype(np.float64) - Cref)
    ok = bool(np.all(err <= 1e-5 * ab))
    return {"value": 2.0 * A.shape[0] * A.shape[1] * B.shape[1] / s / 1e12, "unit": "TFLOP/s",
            "cores": O.max_threads(), "kind": "port",
            "sample": f"C[0:{A.shape[0]}, 0:{B.shape[1]}] of the 32768^3 product (full K), "
                      "oracle/gpcx_oracle.c f32 with every host thread",
            "parity": {"entries": int(C.size), "within_tolerance": ok,
                       "max_err_over_bound": float(np.max(err / np.maximum(1e-5 * ab, 1e-300))),
                       "tolerance": "1e-5 * sum|a||b| vs f64 oracle on bf16-rounded operands"}}


def cpu_demosaic(sample_rows: int = 2048, reps: int = 3) -> dict:
    """The REFERENCE's own demosaic (proj/src/demosaic.cpp, compiled from its
    sources into oracle/_ref) on a row band of the bench mosaic, all host
    cores (ExecPlan workers = nproc)."""
    from oracle import oracle as O
    img = np.random.default_rng(SEED).integers(0, 1 << 16, sample_rows * DM, dtype=np.uint16)
    res = {}
    for name, grad in (("bilinear", False), ("gradient", True)):
        times = []
        for _ in range(reps):
            t = time.perf_counter()
            O.ref_demosaic(grad, img, sample_rows, DM, "RGGB", workers=O.max_threads())
            times.append(time.perf_counter() - t)
        res[name] = sample_rows * DM / statistics.median(times) / 1e9
    return {"value": round(res["bilinear"], 4), "gradient": round(res["gradient"], 4),
            "unit": "Gpixel/s", "cores": O.max_threads(), "kind": "reference",
            "sample": f"BAYER_BILINEAR / BAYER_GRADIENT on a {sample_rows}x{DM} uniform16 mosaic, "
                      f"median of {reps}: the reference's img::demosaic_* with {O.max_threads()} workers"}


def traffic_from_profiles() -> dict:
    p = ROOT / "profiles" / "traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def run_b200(args) -> None:
    import torch
    leg_s: dict[str, float] = {}

    def _leg(name, fn, *a, **k):
        """Runs one leg, adding its wall-clock seconds to `bench_legs_s`."""
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            leg_s[name] = round(leg_s.get(name, 0.0) + time.perf_counter() - t, 2)
    d = Dist(args.gpus)
    d.init("nccl")
    mode = 0
    lut = _leg("lut_device_leg", lut_device_leg, d, args.steps, args.warmup, mode)
    # the other LUT mode (contrast stretch): min/max instead of a histogram
    # at N=1 (read-only reduction, no atomics); the same exchange at N>1
    stretch = _leg("lut_device_leg", lut_device_leg, d, args.steps, args.warmup, 1, gather=False)
    stretch_ms = d.max(stretch["ms"])
    ms = d.max(lut["ms"])
    exch_ms = d.max(lut["exch_ms"]) if lut["exch_ms"] is not None else None
    hist_ms = d.max(lut["hist_ms"])
    gather_ms = d.max(lut["gather_ms"]) if lut["gather_ms"] is not None else None
    # demosaic (HBM-bound, but its gradient kernel is ~90% SM-busy) before the
    # matmul legs: after the 1 kW C4 GEMMs the clock sits at the power cap
    dm = None
    if args.workload in ("all", "demosaic") and d.rank == 0:
        torch.cuda.empty_cache()
        dm = _leg("demosaic_leg", demosaic_leg, max(3, min(args.steps, 10)), 3)
    mm = c4 = c4_tf32 = None
    if args.workload in ("all", "matmul"):
        torch.cuda.empty_cache()
        # C2 before C4: right after the 1 kW C4 GEMMs the power controller
        # still holds the clock down for a while
        if d.rank == 0:
            mm = _leg("matmul_device_leg", matmul_device_leg, max(3, min(args.steps, 10)), 2)
        d.barrier()
        c4 = _leg("matmul_c4_leg", matmul_c4_leg, d, max(2, min(args.steps, 5)), 1)
        # the TF32 tensor-core path on the same C4 problem (kind::tf32)
        c4_tf32 = _leg("matmul_c4_leg", matmul_c4_leg, d, 2, 1, prec=1)
        c4_tf32["ms_max"] = d.max(c4_tf32["ms"])
        c4["ms_max"] = d.max(c4["ms"])
        c4["compute_ms_max"] = d.max(c4["compute_ms"])
        if c4["replicate_ms"] is not None:
            c4["replicate_ms"] = d.max(c4["replicate_ms"])
        if c4["gather_ms"] is not None:
            c4["gather_ms"] = d.max(c4["gather_ms"])
    d.barrier()
    if d.rank != 0:
        d.close()
        return
    d.close()
    pk = peaks()
    px_total = ROWS * COLS
    value = px_total * args.steps / (ms / 1e3) / 1e9
    band_px = lut["band_px"]
    tr = traffic_from_profiles()
    step_ach = 6.0 * band_px / (ms / args.steps / 1e3) / 1e9
    # fused_kernel launches (1 at N=1 and with the peer exchange at N>1;
    # count, then build+apply around the NCCL all-reduce otherwise) carry
    # the step's 6 B/px of algorithmic traffic.
    kern_ms = hist_ms - (exch_ms or 0.0)
    fused_ach = 6.0 * band_px / (kern_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": "lut::fused_kernel", "achieved": round(fused_ach, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(fused_ach / pk["hbm_gbs"], 4),
            "traffic": tr.get("fused_kernel", {}).get("bytes_per_launch_at", {}).get(str(band_px)),
            "algorithmic_bytes_per_launch": 6 * band_px, "peak_source": pk["source"],
            "kernels": {"fused_kernel": {"ms": round(kern_ms, 4),
                                         "phases": "histogram (2 B/px read into a u32 smem window / packed "
                                                   "u16 bins, + 1 B/px residual plane written) | merge + LUT | "
                                                   "apply (1 B/px plane read, 2 B/px written)"},
                        "step": {"achieved": round(step_ach, 1),
                                 "frac": round(step_ach / pk["hbm_gbs"], 4),
                                 "algorithmic_bytes": 6 * band_px}}}
    if exch_ms is not None:
        roof["kernels"]["histogram_all_reduce"] = {"ms": round(exch_ms, 4), "bytes": 262144}
    if lut["exchange"] == "peer":
        roof["kernels"]["fused_kernel"]["phases"] = (
            "histogram (2 B/px read + 1 B/px residual plane written) | publish slice + system-scope "
            "flag rendezvous + P2P sum of the peers' slices | LUT | apply (1 B/px plane read, 2 B/px written)")
    gather = None
    if gather_ms is not None:
        gather = {"ms": round(gather_ms, 3), "bytes": 2 * ROWS * COLS,
                  "what": "corrected bands gathered to rank 0 (exact-size point-to-point receives into the full image, shard.gather_bands; "
                          + ("gloo via host: GPCX_BENCH_ONE_GPU test mode" if Dist.one_gpu else "NCCL")
                          + "); not in `value` -- the output stays sharded in HBM there"}
    launches = 1 if exch_ms is None else 2
    line = {"metric": METRIC, "value": round(value, 2), "unit": "Gpixel/s", "n_gpus": d.n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic (ramp12 splitmix64 scene, generated on device)",
            "config": c3_config(d.n),
            "exchange": (None if d.n == 1 else
                         "65536-bin histogram exchange " + ("fused into the kernel over peer memory "
                                                            "(IPC / NVLink P2P)" if lut["exchange"] == "peer"
                                                            else "by NCCL all-reduce")),
            # per step: fused_kernel once (N=1, or N>1 with the peer exchange);
            # count + build/apply launches with the NCCL exchange
            "roofline": roof, "gpu_launches": launches * args.steps,
            "clocks": lut["clocks"]}
    if gather is not None:
        line["gather"] = gather
    st_ach = 6.0 * band_px / (stretch_ms / args.steps / 1e3) / 1e9
    line["stretch"] = {
        "workload": "C3 with mode=stretch (LUT from the global min/max)",
        "value": round(px_total * args.steps / (stretch_ms / 1e3) / 1e9, 2), "unit": "Gpixel/s",
        "ms_per_step": round(stretch_ms / args.steps, 4),
        "kernels": ("lut::stretch_fused_kernel, one cooperative launch: min/max (2 B/px, redux.sync) "
                    "| grid sync | per-CTA stretch LUT in smem | apply (4 B/px)" if d.n == 1 else "fused_kernel with the peer exchange, as equalize"),
        "roofline": {"bound": "hbm", "achieved": round(st_ach, 1), "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": round(st_ach / pk["hbm_gbs"], 4),
                     "algorithmic_bytes_per_step": 6 * band_px},
        "clocks": stretch["clocks"]}
    # e2e first among the host-heavy legs: the C5 / C1 TCP traffic and the
    # CPU baselines load the host memory system the PCIe copies share
    # the same K requests as the device-timed `value` (a job of K scenes);
    # with 2 in flight the pipeline fill / drain (first H2D, last D2H alone)
    # is amortised over K like any other part of the job
    e2e_steps = max(4, args.steps)
    e2e1 = _leg("lut_e2e_leg", lut_e2e_leg, d.n, e2e_steps, 1, mode, inflight=1)
    e2e2 = _leg("lut_e2e_leg", lut_e2e_leg, d.n, e2e_steps, 1, mode, inflight=2)
    best = e2e2 if e2e2["value"] > e2e1["value"] else e2e1
    line["e2e"] = {"value": round(best["value"], 3), "unit": "Gpixel/s",
                   "h2d_bytes_per_step": best["h2d_bytes_per_step"],
                   "d2h_bytes_per_step": best["d2h_bytes_per_step"],
                   "ms_per_step": round(best["ms_per_step"], 2), "inflight": best["inflight"],
                   "single_request": {"value": round(e2e1["value"], 3),
                                      "ms_per_step": round(e2e1["ms_per_step"], 2)},
                   "path": "gpcx_lut_host (C ABI), pinned host buffers, all N GPUs in-process; "
                           "each step = one full C3 scene in (2 GiB H2D) and out (2 GiB D2H)"}
    c5 = c1 = served = None
    if args.workload in ("all", "c5"):
        time.sleep(2)  # let the clock recover from the C4 leg
        c5 = _leg("c5_leg", c5_leg, d.n)
        c1 = _leg("c1_leg", c1_leg, d.n)
        served = _leg("served_leg", served_leg, d.n, matmul=args.workload == "all")
    if c4 is not None:
        flops = 2.0 * MM4 ** 3
        tf = flops / (c4["ms_max"] / 1e3) / 1e12
        per_gpu_flops = 2.0 * c4["rows"] * MM4 * MM4
        ach = per_gpu_flops / (c4["compute_ms"] / 1e3) / 1e12
        peak = pk["bf16_tflops_sustained"] or pk["bf16_tflops"]
        line["matmul"] = {
            "workload": f"C4: MATMUL prec=bf16 (tcgen05), {MM4}^3, block rows of A/C per GPU, "
                        "B replicated from per-GPU k-slices every step",
            "metric": "matmul TFLOP/s", "value": round(tf, 1), "unit": "TFLOP/s",
            "ms_per_step": round(c4["ms_max"], 3), "scaling": "strong",
            "includes": ("f32->bf16 operand preparation + GEMM + f32 C write"
                         + ("" if d.n == 1 else " + B all-gather (NCCL, side stream, pipelined under "
                                                "the previous step's GEMM)")),
            "compute_ms_per_step": round(c4["compute_ms_max"], 3),
            "b_replicate_ms": None if c4["replicate_ms"] is None else round(c4["replicate_ms"], 3),
            "tolerance": "|c-c_ref| <= 1e-5 * sum|a||b| vs f64 oracle on bf16-rounded operands (tests/test_matmul_gpu.py)",
            "roofline": {"bound": "tensor", "kernel": "gemm::gemm2_kernel<bf16> (+ prep_a/prep_bt)",
                         "achieved": round(ach, 1),
                         "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                         "peak_source": f"{pk['source']} bf16 cuBLAS, sustained (kernel timed in a long loop)",
                         "traffic": tr.get("gemm2_kernel", {}).get("bytes_per_launch")},
            "clocks": c4["clocks"]}
        if c4["gather_ms"] is not None:
            line["matmul"]["gather"] = {"ms": round(c4["gather_ms"], 3), "bytes": 4 * MM4 * MM4,
                                        "what": "C bands (f32) gathered to rank 0, not in `value`"}
        if c4_tf32 is not None:
            tf32 = flops / (c4_tf32["ms_max"] / 1e3) / 1e12
            line["matmul"]["tf32"] = {
                "workload": "C4 with prec=tf32 (tcgen05 kind::tf32, operands rounded RNA)",
                "value": round(tf32, 1), "unit": "TFLOP/s", "ms_per_step": round(c4_tf32["ms_max"], 3),
                "tolerance": "|c-c_ref| <= 1e-5 * sum|a||b| vs f64 oracle on tf32-rounded operands",
                "roofline": {"bound": "tensor", "achieved": round(tf32, 1),
                             "peak": round((pk["bf16_tflops_sustained"] or pk["bf16_tflops"]) / 2, 1),
                             "unit": "TFLOP/s",
                             "peak_note": "half the measured sustained bf16 rate (dense tf32 = 1/2 bf16)",
                             "frac": round(tf32 / ((pk["bf16_tflops_sustained"] or pk["bf16_tflops"]) / 2), 4)},
                "clocks": c4_tf32["clocks"]}
    if mm is not None:
        mm_line = {"workload": "C2: MATMUL prec=f32 (SIMT, reference precision), 4096^3",
                   "value": round(mm["tflops"], 2),
                   "unit": "TFLOP/s", "ms": round(mm["ms"], 3),
                   "roofline": {"bound": "fp32-simt", "kernel": "gemm::sgemm4_kernel (+ transpose_kernel for A^T)",
                                "peak_note": "148 SMs x 128 FFMA x 2 x 1.965 GHz = 74.4 TFLOP/s nominal",
                                "achieved": round(mm["tflops"], 2), "peak": 74.4,
                                "frac": round(mm["tflops"] / 74.4, 4)},
                   "l2": "flushed between steps (256 MiB write)", "clocks": mm["clocks"]}
        mm_line["e2e"] = _leg("matmul_e2e_leg", matmul_e2e_leg, 3)
        line.setdefault("matmul", {})["c2_f32"] = mm_line
    if dm is not None:
        kern = {}
        for name, r in dm.items():
            ach = 8.0 * DM * DM / (r["ms"] / 1e3) / 1e9
            kern[name] = {"ms": round(r["ms"], 4), "value": round(DM * DM / r["ms"] / 1e6, 1),
                          "achieved": round(ach, 1), "frac": round(ach / pk["hbm_gbs"], 4),
                          "clocks": r["clocks"]}
        line["demosaic"] = {
            "workload": f"SURVEY 8f row 1: BAYER_BILINEAR / BAYER_GRADIENT (RGGB), {DM}x{DM} uniform16 "
                        "mosaic on 1 GPU, device-resident",
            "metric": "demosaic Gpixel/s", "value": kern["bilinear"]["value"], "unit": "Gpixel/s",
            "roofline": {"bound": "hbm", "kernel": "demosaic::demosaic_kernel",
                         "algorithmic_bytes_per_launch": 8 * DM * DM, "unit": "GB/s",
                         "peak": pk["hbm_gbs"], "achieved": kern["bilinear"]["achieved"],
                         "frac": kern["bilinear"]["frac"], "traffic": tr.get("demosaic_kernel", {}).get("bytes_per_launch")},
            "kernels": kern, "l2": "inputs + outputs (2 GiB) larger than L2",
            "parity": "byte-identical to the reference's img::demosaic_* and gpcref oracles (tests/test_demosaic.py)"}
        line["demosaic"]["e2e"] = _leg("demosaic_task_leg", demosaic_task_leg)
    # CPU baselines last: their all-core OpenMP runs heat the host and slow
    # the TCP-bound C5 leg if they run before it
    # parity of the timed outputs (equalize and stretch) against the oracle
    # on the whole scene; at N=1 the same oracle runs are the CPU baseline
    lut_ref = _leg("cpu_lut_full", cpu_lut_full, reps=3 if d.n == 1 else 1)
    line["parity"] = {"equalize": lut_parity(lut, lut_ref[0]), "stretch": lut_parity(stretch, lut_ref[1])}
    line["parity"]["ok"] = line["parity"]["equalize"]["ok"] and line["parity"]["stretch"]["ok"]
    line["stretch"]["parity"] = line["parity"]["stretch"]["ok"]
    if d.n == 1:
        line["cpu_baseline"] = cpu_lut(lut_ref, mode)
        line["stretch"]["cpu_baseline"] = cpu_lut(lut_ref, 1)
        if mm is not None:
            line["matmul"]["c2_f32"]["cpu_baseline"] = _leg("cpu_matmul", cpu_matmul)
        if dm is not None:
            line["demosaic"]["cpu_baseline"] = _leg("cpu_demosaic", cpu_demosaic)
        if c4 is not None and c4.get("sample") is not None:
            line["matmul"]["cpu_baseline"] = _leg("cpu_matmul_c4", cpu_matmul_c4, c4["sample"])
    if c5 is not None:
        if d.n == 1:
            c5["cpu_baseline"] = _leg("cpu_c5", cpu_c5)
        line["c5"] = c5
    if c1 is not None:
        if d.n == 1:
            ref = _leg("cpu_c1", cpu_c1)
            c1["cpu_baseline"] = ref
            c1["output_identical_to_reference_server"] = ref.pop("digest") == c1["digest"]
        c1.pop("digest")
        line["c1"] = c1
    if served is not None:
        served["c3"]["parity"] = served["c3"].pop("digest") == lut_ref[0]["digest"]
        served["workload"] = ("C3 / C4 through the B200 server as header-only requests (synth=, SURVEY 8d "
                              "option ii): inputs generated on the GPUs, native client, loopback TCP")
        line["served"] = served
    line["bench_legs_s"] = leg_s
    print(json.dumps(line), flush=True)


def run_reference(args) -> None:
    """The reference arm: the restated CPU path (oracle/gpcx_oracle.c; the
    reference has no LUT / matmul implementation to install, SURVEY.md
    §0.3) on the box's host cores, on the SAME workload as the B200 arm --
    LUT_CORRECT equalize of the whole 32768^2 C3 scene per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # every host core, explicitly: torchrun exports OMP_NUM_THREADS=1 (N>1),
    # and libgomp reads it when the oracle library is loaded
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    from oracle import oracle as O
    mode = 0
    img = O.synth_image(O.IMG_RAMP12, SEED, ROWS, COLS)
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        out, _, st = O.lut_correct(img, mode, threads=cores)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    dig = O.digest_u16(out)
    px = ROWS * COLS
    value = px * len(times) / sum(times) / 1e9
    sample = (f"LUT_CORRECT equalize of the whole {ROWS}x{COLS} C3 scene per step (no sampling), "
              f"oracle/gpcx_oracle.c (restatement; the reference has no LUT code), {cores} OpenMP threads")
    line = {"metric": METRIC, "value": round(value, 4), "unit": "Gpixel/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": c3_config(args.gpus),
            "output": {"digest": f"{dig:016x}", "stats": st},
            "cpu_baseline": {"value": round(value, 4), "unit": "Gpixel/s", "cores": cores,
                             "kind": "port", "sample": sample, "host": O.host_cpu()},
            "e2e": {"value": round(value, 4), "unit": "Gpixel/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------- gpc bench, GPU columns ---

def _median_ms(run, reps: int = 5) -> float:
    """gpc.cpp:243-254: median of 5 wall-clock runs."""
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        run()
        ts.append((time.perf_counter() - t) * 1e3)
    return sorted(ts)[len(ts) // 2]


def _gpu_median_ms(run, reps: int = 5) -> float:
    import torch
    run()  # warm-up (lazy allocations, attributes)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def run_gpc_bench(args) -> None:
    """`gpc bench` (proj/tools/gpc.cpp:256-370) with the GPU columns SURVEY.md
    §8 a12 asks for: per task and worker count the reference's serial and
    parallel CPU times (the reference's own kernels from oracle/_ref for
    BAYER_*, the restated oracle for LUT_CORRECT / MATMUL), then the B200
    kernel on one GPU (device-resident, CUDA events, median of 5), its
    throughput and roofline fraction.  TSV on stdout."""
    import torch
    from oracle import oracle as O
    from paper_1505_05655_b200 import device as D
    pk = peaks()
    task = args.task
    hw = len(os.sched_getaffinity(0))
    workers = [int(w) for w in (args.workers_list or f"1,{hw}").split(",")]
    cols = ["task", "config", "workers", "serial_ms", "parallel_ms", "speedup", "gpus", "gpu_ms",
            "gpu_speedup", "throughput", "unit", "roofline_frac"]
    print("\t".join(cols))
    rng = np.random.default_rng(0x5EED)

    def row(config, w, serial, parallel, gpu_ms, thr, unit, frac):
        print("\t".join([task, config, str(w), f"{serial:.3f}", f"{parallel:.3f}",
                         f"{serial / parallel:.2f}", "1", f"{gpu_ms:.4f}", f"{serial / gpu_ms:.1f}",
                         f"{thr:.2f}", unit, f"{frac:.3f}"]), flush=True)

    if task in ("BAYER_BILINEAR", "BAYER_GRADIENT"):
        rows, cols_ = (int(x) for x in (args.dims or "2048x2048").split("x"))
        grad = task == "BAYER_GRADIENT"
        img = rng.integers(0, 1 << 16, rows * cols_, dtype=np.uint16)
        serial = _median_ms(lambda: O.ref_demosaic(grad, img, rows, cols_, gpcref=True))
        dimg = torch.from_numpy(img.view(np.int16)).cuda()
        out = torch.empty(3 * rows * cols_, dtype=torch.int16, device="cuda")
        gms = _gpu_median_ms(lambda: D.demosaic(grad, 0, dimg, rows, cols_, out))
        thr = rows * cols_ / gms / 1e6
        frac = 8.0 * rows * cols_ / (gms / 1e3) / 1e9 / pk["hbm_gbs"]
        for w in workers:
            par = _median_ms(lambda: O.ref_demosaic(grad, img, rows, cols_, workers=w))
            row(f"{rows}x{cols_}", w, serial, par, gms, thr, "Gpixel/s", frac)
    elif task == "LUT_CORRECT":
        rows, cols_ = (int(x) for x in (args.dims or "4096x4096").split("x"))
        img = O.synth_image(O.IMG_RAMP12, SEED, rows, cols_)
        serial = _median_ms(lambda: O.lut_correct(img, O.LUT_EQUALIZE, threads=1))
        dimg = D.synth_image(0, SEED, rows, cols_)
        out = torch.empty_like(dimg)
        lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(dimg.numel())
        gms = _gpu_median_ms(lambda: D.lut_correct(dimg, out, O.LUT_EQUALIZE, lut, stats, ws))
        thr = rows * cols_ / gms / 1e6
        frac = 6.0 * rows * cols_ / (gms / 1e3) / 1e9 / pk["hbm_gbs"]
        for w in workers:
            par = _median_ms(lambda: O.lut_correct(img, O.LUT_EQUALIZE, threads=w))
            row(f"{rows}x{cols_}/equalize", w, serial, par, gms, thr, "Gpixel/s", frac)
    elif task == "MATMUL":
        m = k = n = int(args.dims or 1024)
        A = O.synth_matrix(O.MAT_UNIFORM32, SEED, m, k)
        B = O.synth_matrix(O.MAT_UNIFORM32, SEED_B, k, n)
        serial = _median_ms(lambda: O.matmul_f32(A, B, threads=1), reps=3)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.empty(m, n, device="cuda")
        for prec, name in ((0, "f32"), (2, "bf16")):
            ws = D.matmul_workspace(prec, m, n, k)
            gms = _gpu_median_ms(lambda: D.matmul(prec, dA, dB, dC, ws))
            tf = 2.0 * m * n * k / gms / 1e9
            peak = 74.4 if prec == 0 else (pk["bf16_tflops_sustained"] or pk["bf16_tflops"])
            for w in workers:
                par = _median_ms(lambda: O.matmul_f32(A, B, threads=w), reps=3)
                row(f"{m}^3/prec={name}", w, serial, par, gms, tf, "TFLOP/s", tf / peak)
    else:
        raise SystemExit("--task must be BAYER_BILINEAR, BAYER_GRADIENT, LUT_CORRECT or MATMUL")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=["all", "lut", "matmul", "c5", "demosaic"], default="all")
    # `gpc bench` mode (TSV, proj/tools/gpc.cpp:256-370 + GPU columns)
    ap.add_argument("--gpc-bench", action="store_true")
    ap.add_argument("--task", default="LUT_CORRECT")
    ap.add_argument("--dims", default="")
    ap.add_argument("--workers-list", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpc_bench:
        run_gpc_bench(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
