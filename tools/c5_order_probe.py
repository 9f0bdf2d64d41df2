import sys, json, time
sys.path.insert(0, '.')
import bench
def c5(tag):
    r = bench.c5_leg(1); print(tag, json.dumps({"chains_per_s": round(r["chains_per_s"], 1)}), flush=True)
c5("c5 first")
e1 = bench.lut_e2e_leg(1, 20, 1, 0, inflight=1); e2 = bench.lut_e2e_leg(1, 20, 1, 0, inflight=2)
print("e2e", round(e2["value"], 2), flush=True)
c5("c5 after e2e")
time.sleep(5)
c5("c5 after e2e + 5 s")
