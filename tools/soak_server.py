"""Soak of the B200 server: C5 passes (64 concurrent clients x LUT_GEN ->
LUT_APPLY -> MATMUL bf16) interleaved with header-only C3 requests and
malformed frames, for a fixed wall time; prints per pass the chains/s, the
server's request / error counters, the process RSS and the device memory in
use -- all must stay flat (no leak of slots, pinned buffers or sockets).

    python tools/soak_server.py [seconds]
"""
import json, os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import psutil
import torch
import bench
import paper_1505_05655_b200 as G
from paper_1505_05655_b200.client import submit_native as submit

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120
imgs, B = bench.c5_inputs()
proc = psutil.Process()
G.init([0])
with G.Server(max_tasks=0) as srv:
    t0 = time.time()
    p = 0
    while time.time() - t0 < secs:
        r = bench.c5_run(srv.port, imgs, B, "bf16")
        q = submit("127.0.0.1", srv.port, "LUT_CORRECT",
                   "rows=8192,cols=8192,mode=equalize,synth=ramp12,seed=7", [], resp_cap=64)
        with socket.create_connection(("127.0.0.1", srv.port)) as s:  # a malformed frame
            s.sendall(b"\xff" * 260)
            s.settimeout(10)
            try:
                s.recv(260)
            except OSError:
                pass
        free, total = torch.cuda.mem_get_info()
        st = srv.stats()
        print(json.dumps({"pass": p, "t": round(time.time() - t0, 1), "chains_per_s": round(r["chains_per_s"], 1),
                          "synth_ok": q.ok, "requests": st.get("requests"), "busy": st.get("busy"),
                          "dropped": st.get("dropped"), "rss_MB": proc.memory_info().rss >> 20,
                          "dev_used_MB": (total - free) >> 20, "fds": proc.num_fds()}), flush=True)
        p += 1
