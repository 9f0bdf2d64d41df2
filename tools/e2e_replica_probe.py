"""The C3 e2e pattern rebuilt on the device-level API (torch copies +
gpcx_lut_correct_device / gpcx_lut_apply_device), 2 threads in flight --
to split gpcx_lut_host's cost into copy pattern, kernel and host code."""
import json, os, sys, threading as th, time
sys.path.insert(0, '.')
import torch
from paper_1505_05655_b200 import device as D
n = 32768 * 32768
def run(kind, inflight=2, per=6):
    ctx = []
    for _ in range(inflight):
        h_in = torch.full((n,), 7, dtype=torch.int16).pin_memory(); h_out = torch.empty(n, dtype=torch.int16).pin_memory()
        d_in = torch.empty(n, dtype=torch.int16, device="cuda"); d_out = torch.empty_like(d_in)
        ctx.append((h_in, h_out, d_in, d_out, D.new_lut(), D.new_stats(), D.lut_workspace(n), torch.cuda.Stream()))
    phases = []
    launch_ms = []
    def one(c):
        h_in, h_out, d_in, d_out, lut, stats, ws, s = c
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            d_in.copy_(h_in, non_blocking=True)
            ev[1].record(s)
            if kind == "correct_sync":
                s.synchronize()  # H2D done before the cooperative launch is queued
                D.lut_correct(d_in, d_out, 0, lut, stats, ws, s)
            if kind == "correct":
                t_l = time.perf_counter()
                D.lut_correct(d_in, d_out, 0, lut, stats, ws, s)
                launch_ms.append((time.perf_counter() - t_l) * 1e3)
            elif kind == "stretch":
                D.lut_correct(d_in, d_out, 1, lut, stats, ws, s)
            elif kind == "apply":
                D.lut_apply(lut, d_in, d_out, s)
            ev[2].record(s)
            h_out.copy_(d_out if kind != "copy" else d_in, non_blocking=True)
            ev[3].record(s)
            s.synchronize()
        phases.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
    def worker(k, count):
        for _ in range(count):
            one(ctx[k])
    ws_ = [th.Thread(target=worker, args=(k, 1)) for k in range(inflight)]; [w.start() for w in ws_]; [w.join() for w in ws_]
    t = time.perf_counter()
    ws_ = [th.Thread(target=worker, args=(k, per)) for k in range(inflight)]; [w.start() for w in ws_]; [w.join() for w in ws_]
    ms = round(1e3 * (time.perf_counter() - t) / (per * inflight), 2)
    ph = phases[inflight:]
    avg = [round(sum(p[i] for p in ph) / len(ph), 2) for i in range(3)]
    out = {"ms_per_request": ms, "h2d_kernel_d2h_ms": avg}
    if launch_ms:
        out["host_launch_ms"] = [round(x, 2) for x in sorted(launch_ms)[::3]]
    return out
INFLIGHT = int(os.environ.get("INFLIGHT", "2"))
for kind in sys.argv[1:] or ("copy", "apply", "correct", "copy", "apply", "correct"):
    print(json.dumps({kind: run(kind, INFLIGHT)}), flush=True)
