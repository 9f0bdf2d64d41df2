"""Test configuration.

Markers: `gpu` -- needs a CUDA device (run with -m gpu on a B200).  The CPU
suite (-m "not gpu") covers the oracle against its KATs / golden vectors,
the host-side logic, the wire / dispatch behaviour against the compiled
reference, and that libgpcx.so loads and exports include/gpcx.h.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
os.environ.setdefault("GPCX_QUIET", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    lib = ROOT / "paper_1505_05655_b200" / "lib" / "libgpcx.so"
    if not lib.exists():  # build container only; the GPU box gets the prebuilt .so
        import runpy
        runpy.run_path(str(ROOT / "paper_1505_05655_b200" / "build.py"), run_name="build_only")["build"]()


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("this test needs a CUDA device (run -m gpu on a B200 box)")
    import torch
    torch.cuda.init()
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def refl():
    from oracle import oracle as O
    if O.ref is None:
        pytest.skip("oracle/_ref/libgpc_ref.so not built (needs /root/reference at build time)")
    return O
