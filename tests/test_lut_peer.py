"""Row-band LUT_CORRECT with the histogram exchange fused into the kernel
over peer memory (gpcx_lut_peer_*, one process per rank).

On the 1-GPU test box every rank is a separate process on cuda:0: the IPC
mappings are then second mappings of the same HBM and the ranks' kernels
meet through time-slicing, which exercises the whole protocol (publish,
system-scope flags, double-buffered histograms, P2P sums) except NVLink
itself.  Results must equal the single-device oracle bit for bit, on every
rank and every step."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def shared_gpu(gpu):
    """The ranks are separate processes on cuda:0: needs the Default compute
    mode (an exclusive-process GPU admits one context)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        mode = pynvml.nvmlDeviceGetComputeMode(pynvml.nvmlDeviceGetHandleByIndex(0))
        pynvml.nvmlShutdown()
    except Exception:
        return gpu
    if mode != 0:  # NVML_COMPUTEMODE_DEFAULT
        pytest.skip(f"compute mode {mode}: one process per GPU only")
    return gpu

_WORKER = r"""
import json, os, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, os.environ["GPCX_ROOT"])
from paper_1505_05655_b200 import device as D
rank, nranks, tmp = int(sys.argv[1]), int(sys.argv[2]), Path(sys.argv[3])
rows, cols, kind, seed, steps = (int(x) for x in sys.argv[4:9])
modes = [int(m) for m in sys.argv[9].split(",")]
torch.cuda.set_device(0)
per = (rows + nranks - 1) // nranks
r0 = min(rows, rank * per); nr = min(per, rows - r0)
img = D.synth_image(kind, seed, rows, cols, r0, nr)
out = torch.empty_like(img)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(max(1, img.numel()))
p = D.LutPeer(rank, nranks)
(tmp / f"h{rank}.tmp").write_bytes(p.handle()); os.replace(tmp / f"h{rank}.tmp", tmp / f"h{rank}.bin")
t0 = time.time()
while not all((tmp / f"h{r}.bin").exists() for r in range(nranks)):
    if time.time() - t0 > 60: raise SystemExit("peers never published their handles")
    time.sleep(0.01)
p.connect([(tmp / f"h{r}.bin").read_bytes() for r in range(nranks)])
res = []
for step in range(steps):
    mode = modes[step % len(modes)]
    out.zero_()
    p.correct(img, out, mode, lut, stats, ws)
    torch.cuda.synchronize()
    dig = int(D.digest_u16(out, r0 * cols).item()) & (2**64 - 1)
    res.append({"mode": mode, "digest": dig, "stats": D.read_stats(stats),
                "lut": lut.cpu().numpy().view(np.uint16).tobytes().hex()})
    np.save(tmp / f"out{rank}_{step}.npy", out.cpu().numpy().view(np.uint16))
(tmp / f"res{rank}.json").write_text(json.dumps(res))
p.close()
"""


def _run_group(tmp_path, nranks, rows, cols, kind, seed, steps, modes):
    env = dict(os.environ, GPCX_ROOT=str(ROOT), GPCX_PEER_TIMEOUT_MS="30000")
    procs = [subprocess.Popen([sys.executable, "-c", _WORKER, str(r), str(nranks), str(tmp_path),
                               str(rows), str(cols), str(kind), str(seed), str(steps),
                               ",".join(map(str, modes))],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(nranks)]
    errs = []
    for p in procs:
        try:
            _, err = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            _, err = p.communicate()
        if p.returncode != 0:
            errs.append(err[-3000:])
    assert not errs, "\n".join(errs)
    return [json.loads((tmp_path / f"res{r}.json").read_text()) for r in range(nranks)]


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,rows,cols,kind", [
    (2, 1000, 777, 0),     # ragged band sizes, odd row length
    (2, 4096, 4096, 1),    # uniform16: every bin populated
    (3, 2049, 1024, 0),    # three ranks, uneven split
    (3, 2, 5, 1),          # rank 2's band is empty: it still meets its peers
    (2, 8192, 8200, 0),    # bands >= 2^25 samples: the residual plane in the peer launch
])
def test_peer_exchange_equals_single_device_oracle(shared_gpu, tmp_path, nranks, rows, cols, kind):
    from oracle import oracle as O
    steps, modes = 4, [O.LUT_EQUALIZE, O.LUT_EQUALIZE, O.LUT_STRETCH, O.LUT_EQUALIZE]
    res = _run_group(tmp_path, nranks, rows, cols, kind, 0x5EED, steps, modes)
    whole = O.synth_image(kind, 0x5EED, rows, cols).ravel()
    per = (rows + nranks - 1) // nranks
    for step in range(steps):
        mode = modes[step]
        ref_out, ref_lut, ref_st = O.lut_correct(whole, mode)
        got = np.concatenate([np.load(tmp_path / f"out{r}_{step}.npy") for r in range(nranks)])
        assert np.array_equal(got, ref_out), (step, mode)
        for r in range(nranks):
            rr = res[r][step]
            assert bytes.fromhex(rr["lut"]) == ref_lut.tobytes(), (step, r)
            assert rr["stats"] == ref_st, (step, r, rr["stats"], ref_st)
        assert sum(min(per, max(0, rows - r * per)) for r in range(nranks)) == rows


_BIG_WORKER = r"""
import json, os, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, os.environ["GPCX_ROOT"])
from paper_1505_05655_b200 import device as D
rank, tmp, n, bulk = int(sys.argv[1]), Path(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
torch.cuda.set_device(0)
# band: values 0..65535 once, then `bulk` for the remaining n - 65536 samples
img = torch.full((n,), bulk, dtype=torch.int32, device="cuda").to(torch.int16)
img[:65536] = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.int16)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(n)
p = D.LutPeer(rank, 2)
(tmp / f"h{rank}.tmp").write_bytes(p.handle()); os.replace(tmp / f"h{rank}.tmp", tmp / f"h{rank}.bin")
t0 = time.time()
while not all((tmp / f"h{r}.bin").exists() for r in range(2)):
    if time.time() - t0 > 60: raise SystemExit("peers never published their handles")
    time.sleep(0.01)
p.connect([(tmp / f"h{r}.bin").read_bytes() for r in range(2)])
res = []
for mode in (0, 1):
    p.correct(img, img, mode, lut, stats, ws)   # in place
    torch.cuda.synchronize()
    l = lut.cpu().numpy().view(np.uint16)
    # out = LUT[in] on the device, checked against the LUT the kernel built
    head = img[:65536].cpu().numpy().view(np.uint16)
    tail_ok = bool((img[65536:] == int(np.int16(np.uint16(l[bulk])))).all().item())
    res.append({"stats": D.read_stats(stats), "lut": l.tobytes().hex(),
                "head_ok": bool(np.array_equal(head, l)), "tail_ok": tail_ok})
    # restore the band for the next mode
    img.fill_(int(np.int16(np.uint16(bulk))))
    img[:65536] = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.int16)
(tmp / f"res{rank}.json").write_text(json.dumps(res))
p.close()
"""


@pytest.mark.gpu
@pytest.mark.slow
def test_peer_group_total_above_2_pow_32(shared_gpu, tmp_path):
    """Two ranks of 2^31 + 2^20 samples each: the group's image holds more
    than 2^32 pixels and one bin alone more than 2^32 counts, so the summed
    histogram, its totals, cdf_min and stats.n must be 64-bit (each band's
    own histogram is u32).  LUT and stats equal the oracle's from the exact
    u64 group histogram; out == LUT[in] on every sample."""
    from oracle import oracle as O
    n, bulk = (1 << 31) + (1 << 20), 30000
    env = dict(os.environ, GPCX_ROOT=str(ROOT), GPCX_PEER_TIMEOUT_MS="60000")
    procs = [subprocess.Popen([sys.executable, "-c", _BIG_WORKER, str(r), str(tmp_path), str(n), str(bulk)],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    errs = []
    for p in procs:
        try:
            _, err = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            _, err = p.communicate()
        if p.returncode != 0:
            errs.append(err[-3000:])
    assert not errs, "\n".join(errs)
    hist = np.full(65536, 2, dtype=np.uint64)
    hist[bulk] += 2 * (n - 65536)
    assert hist[bulk] > 2 ** 32 and hist.sum() > 2 ** 32
    for r in range(2):
        res = json.loads((tmp_path / f"res{r}.json").read_text())
        for mode, rr in zip((O.LUT_EQUALIZE, O.LUT_STRETCH), res):
            ref_lut, ref_st = O.lut_from_hist(hist, mode)
            assert rr["stats"] == ref_st, (r, mode, rr["stats"], ref_st)
            assert bytes.fromhex(rr["lut"]) == ref_lut.tobytes(), (r, mode)
            assert rr["head_ok"] and rr["tail_ok"], (r, mode)


_SILENT_PEER = r"""
import os, sys, time
from pathlib import Path
sys.path.insert(0, os.environ["GPCX_ROOT"])
import torch
from paper_1505_05655_b200 import device as D
rank, tmp = int(sys.argv[1]), Path(sys.argv[2])
torch.cuda.set_device(0)
p = D.LutPeer(rank, 2)
(tmp / f"h{rank}.tmp").write_bytes(p.handle()); os.replace(tmp / f"h{rank}.tmp", tmp / f"h{rank}.bin")
t0 = time.time()
while not (tmp / f"h{1 - rank}.bin").exists():
    if time.time() - t0 > 60: os._exit(3)
    time.sleep(0.01)
p.connect([(tmp / f"h{r}.bin").read_bytes() for r in range(2)])
if rank == 1:   # connected but never launches; stays mapped until rank 0 is done
    while not (tmp / "done").exists() and time.time() - t0 < 120:
        time.sleep(0.05)
    os._exit(0)
img = D.synth_image(0, 1, 64, 64)
out = torch.empty_like(img)
lut, stats, ws = D.new_lut(), D.new_stats(), D.lut_workspace(img.numel())
p.correct(img, out, 0, lut, stats, ws)
try:
    torch.cuda.synchronize()
    print("NO TRAP")
    code = 1
except Exception as e:
    print("TRAPPED", type(e).__name__, str(e)[:120])
    code = 0
(tmp / "done").write_text("x")
sys.stdout.flush()
os._exit(code)
"""


@pytest.mark.gpu
def test_peer_rank_without_peers_traps_instead_of_hanging(shared_gpu, tmp_path):
    """A group of 2 where rank 1 connects but never launches: rank 0's
    kernel must trap after GPCX_PEER_TIMEOUT_MS and the failure must surface
    on its stream (a dead peer never hangs the GPU)."""
    env = dict(os.environ, GPCX_ROOT=str(ROOT), GPCX_PEER_TIMEOUT_MS="2000")
    procs = [subprocess.Popen([sys.executable, "-c", _SILENT_PEER, str(r), str(tmp_path)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=180))
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate())
    assert procs[0].returncode == 0 and "TRAPPED" in outs[0][0], outs[0][0] + outs[0][1][-2000:]
    assert procs[1].returncode == 0, outs[1][1][-2000:]


def test_peer_group_arguments_validated():
    import paper_1505_05655_b200 as G
    import ctypes as C
    p = C.c_void_p(None)
    for rank, nranks in [(0, 0), (2, 2), (-1, 2), (0, 9)]:
        st = G.lib.gpcx_lut_peer_create(rank, nranks, C.byref(p))
        assert st == G.STATUS["BadValue"] or st == G.STATUS["TaskFailed"], (rank, nranks, st)
    assert G.lib.gpcx_lut_peer_connect(None, None) == G.STATUS["BadValue"]
    assert G.lib.gpcx_lut_correct_peer_device(None, None, None, 0, 0, None, None, None, 0,
                                              None) == G.STATUS["BadValue"]
