"""C3 e2e through gpcx_lut_host per op (LUT_CORRECT: cooperative fused
kernel; LUT_APPLY: the plain apply kernel; both move 2 GiB each way), 2 in
flight, 12 requests -- does the cooperative launch cost overlap?"""
import ctypes as C, json, sys, threading as th, time
sys.path.insert(0, '.')
import numpy as np
import paper_1505_05655_b200 as G
ROWS = COLS = 32768
n = ROWS * COLS
lut = np.arange(65536, dtype=np.uint16)
def run(op, inflight=2, per=6):
    bufs = [(G.lib.gpcx_pinned_alloc(n * 2), G.lib.gpcx_pinned_alloc(n * 2)) for _ in range(inflight)]
    for p_in, _ in bufs:
        np.ctypeslib.as_array((C.c_uint16 * n).from_address(p_in))[:] = 7
    def one(p_in, p_out):
        st = G.LutStats()
        G.check(G.lib.gpcx_lut_host(op, 0, ROWS, COLS, C.c_void_p(p_in),
                                    lut.ctypes.data if op == 1 else None, C.c_void_p(p_out), None, C.byref(st)))
    def worker(k, count):
        for _ in range(count):
            one(*bufs[k])
    ws = [th.Thread(target=worker, args=(k, 1)) for k in range(inflight)]; [w.start() for w in ws]; [w.join() for w in ws]
    t = time.perf_counter()
    ws = [th.Thread(target=worker, args=(k, per)) for k in range(inflight)]; [w.start() for w in ws]; [w.join() for w in ws]
    wall = time.perf_counter() - t
    for p_in, p_out in bufs:
        G.lib.gpcx_pinned_free(p_in); G.lib.gpcx_pinned_free(p_out)
    return 1e3 * wall / (per * inflight)
for op, name in ((2, "LUT_CORRECT"), (1, "LUT_APPLY"), (2, "LUT_CORRECT"), (1, "LUT_APPLY")):
    print(json.dumps({"op": name, "ms_per_request": round(run(op), 2)}), flush=True)
