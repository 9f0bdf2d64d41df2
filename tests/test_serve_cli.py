"""`gpcx-serve`, the process entry point (the reference CLI's `gpc serve`,
proj/tools/gpc.cpp:94-128): flags, banner, SIGINT/SIGTERM drain, and a
request served end to end by the reference client."""
from __future__ import annotations

import re
import signal
import subprocess
from pathlib import Path

import numpy as np
import pytest

BIN = Path(__file__).resolve().parent.parent / "paper_1505_05655_b200" / "lib" / "gpcx-serve"


def test_usage_and_bad_flags():
    assert BIN.exists()
    r = subprocess.run([str(BIN), "--help"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "usage:" in r.stderr
    for bad in (["--port", "99999"], ["--max-tasks", "x"], ["--devices", "0,a"], ["--nope", "1"],
                ["--port"]):
        r = subprocess.run([str(BIN), *bad], capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and "usage:" in r.stderr, bad


def test_no_gpu_fails_loudly():
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("a GPU is present")
    r = subprocess.run([str(BIN), "--port", "0"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and r.stderr.startswith("gpcx-serve:")


@pytest.mark.gpu
@pytest.mark.parametrize("sig", [signal.SIGTERM, signal.SIGINT])
def test_serves_then_drains_on_signal(gpu, refl, sig):
    from oracle import oracle as O
    p = subprocess.Popen([str(BIN), "--bind", "127.0.0.1", "--port", "0", "--max-tasks", "4",
                          "--devices", "0"], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                         text=True)
    try:
        banner = p.stdout.readline()
        m = re.match(r"gpcx server listening on 127\.0\.0\.1:(\d+) \(devices=1, max_tasks=4", banner)
        assert m, banner
        port = int(m.group(1))
        img = O.synth_image(O.IMG_RAMP12, 3, 300, 500)
        status, params, data, name = refl.ref_submit(port, "LUT_CORRECT", "rows=300,cols=500",
                                                     img.tobytes(), "c.raw")
        assert status == "OK" and name == "c.raw"
        ref_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
        assert np.frombuffer(data, dtype=np.uint16).tobytes() == ref_out.tobytes()
        p.send_signal(sig)
        _, err = p.communicate(timeout=60)
        assert p.returncode == 0 and f"signal {int(sig)}, draining" in err
    finally:
        if p.poll() is None:
            p.kill()
            p.communicate()


@pytest.mark.gpu
def test_gpc_bench_mode_prints_reference_columns_plus_gpu(gpu, refl):
    """bench.py --gpc-bench: `gpc bench`'s TSV (task, config, workers,
    serial_ms, parallel_ms, speedup; proj/tools/gpc.cpp:256-370) extended
    with gpus, gpu_ms, gpu_speedup, throughput, unit, roofline_frac."""
    import sys
    root = BIN.parent.parent.parent
    for task, dims in (("LUT_CORRECT", "512x768"), ("BAYER_GRADIENT", "256x256"), ("MATMUL", "256")):
        r = subprocess.run([sys.executable, "bench.py", "--gpc-bench", "--task", task, "--dims", dims,
                            "--workers-list", "1,2"], cwd=root, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [l.split("\t") for l in r.stdout.strip().splitlines()]
        assert lines[0] == ["task", "config", "workers", "serial_ms", "parallel_ms", "speedup",
                            "gpus", "gpu_ms", "gpu_speedup", "throughput", "unit", "roofline_frac"]
        assert len(lines) == 1 + (4 if task == "MATMUL" else 2)
        assert all(l[0] == task and float(l[7]) > 0 for l in lines[1:])
