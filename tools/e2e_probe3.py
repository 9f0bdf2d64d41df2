import sys, json
sys.path.insert(0, '.')
import bench
for k in (2, 3, 2, 3):
    r = bench.lut_e2e_leg(1, 20, 1, 0, inflight=k)
    print(k, json.dumps({"ms": round(r["ms_per_step"], 2), "value": round(r["value"], 2)}), flush=True)
