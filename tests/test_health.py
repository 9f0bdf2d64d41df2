"""Device health: a sticky CUDA error quarantines the device, requests
route to the remaining bound devices, and only with none left do GPU tasks
answer ERR:TASK_FAILED (the reference's failure boundary is the handler
exception -> TASK_FAILED, proj/src/registry.cpp:113-118).

On the 1-GPU box "several devices" are bound indices on cuda:0 (G.init([0,
0])), so routing is exercised with the host-side quarantine (fault kind 0);
the real sticky error (fault kind 1: a kernel that traps) poisons the
whole process's context and runs in a subprocess server."""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

import paper_1505_05655_b200 as G

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_quarantined_index_gets_no_work(gpu, refl):
    from oracle import oracle as O
    rows, cols = 4096, 4096  # large enough for the planner to shard over 2 bands
    img = O.synth_image(O.IMG_RAMP12, 3, rows, cols)
    want, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
    try:
        G.init([0, 0])
        assert G.device_health(0) == (True, "") and G.device_health(1) == (True, "")
        G.check(G.lib.gpcx_debug_fault(0, 0))
        ok, why = G.device_health(0)
        assert not ok and why == "gpcx_debug_fault"
        assert G.device_health(1)[0]
        # direct calls and the server both keep working on index 1
        _, out = G.run("LUT_CORRECT", f"rows={rows},cols={cols}", img)
        assert np.array_equal(out.view(np.uint16), want)
        with G.Server(max_tasks=4) as s:
            st, _, data, _ = refl.ref_submit(s.port, "LUT_CORRECT", f"rows={rows},cols={cols}",
                                             img.tobytes())
            assert st == "OK" and data == want.tobytes()
            # the last healthy index goes: GPU tasks fail, device-free ones do not
            G.check(G.lib.gpcx_debug_fault(1, 0))
            st, params, _, _ = refl.ref_submit(s.port, "LUT_CORRECT", "rows=64,cols=64",
                                               img[:4096].tobytes())
            assert st == "ERR:TASK_FAILED" and "no healthy device" in params
            st, _, xml, _ = refl.ref_submit(s.port, "DEVINFO", "", b"")
            assert st == "OK" and b"<gpgpu_server" in xml
        with pytest.raises(G.GpcxError) as e:
            G.run("LUT_CORRECT", "rows=64,cols=64", img[:4096])
        assert e.value.code == "TaskFailed" and "no healthy device" in str(e.value)
        G.init([0, 0])  # rebinding admits the devices again
        assert G.device_health(0)[0] and G.device_health(1)[0]
        _, out = G.run("LUT_CORRECT", "rows=64,cols=64", img[:4096])
    finally:
        G.init([0])


_TRAP_SERVER = textwrap.dedent(r"""
    import os, sys
    sys.path.insert(0, os.environ["GPCX_ROOT"])
    import numpy as np
    import paper_1505_05655_b200 as G
    from oracle import oracle as O
    G.init([0])
    img = O.synth_image(O.IMG_RAMP12, 1, 64, 64)
    with G.Server(max_tasks=2) as s:
        st, _, _, _ = O.ref_submit(s.port, "LUT_CORRECT", "rows=64,cols=64", img.tobytes())
        print("before", st)
        O.ref_submit(s.port, "DEVINFO", "", b"")  # probed (and cached) while healthy
        try:
            G.check(G.lib.gpcx_debug_fault(0, 1))
            print("fault: no error")
        except G.GpcxError as e:
            print("fault", e.code)
        ok, why = G.device_health(0)
        print("health", ok, why.split(" at ")[0])
        for i in range(3):  # answered promptly, never hangs, never touches the dead context
            st, params, _, _ = O.ref_submit(s.port, "LUT_CORRECT", "rows=64,cols=64", img.tobytes())
            print("after", st, "no healthy device" in params)
        st, _, xml, _ = O.ref_submit(s.port, "DEVINFO", "", b"")
        print("devinfo", st)
    print("stopped")
""")


def test_sticky_trap_quarantines_device_in_a_server_process(gpu, refl):
    env = dict(os.environ, GPCX_ROOT=str(ROOT), GPCX_QUIET="1")
    p = subprocess.run([sys.executable, "-c", _TRAP_SERVER], env=env, capture_output=True, text=True,
                       timeout=180)
    out = p.stdout.splitlines()
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    assert "before OK" in out
    assert "fault TaskFailed" in out
    assert "health False cudaErrorLaunchFailure" in out, out
    assert out.count("after ERR:TASK_FAILED True") == 3, out
    assert "devinfo OK" in out and out[-1] == "stopped"
