import sys, json
sys.path.insert(0, '.')
import bench
for k in (1, 2, 3, 4):
    r = bench.lut_e2e_leg(1, 8, 1, 0, inflight=k)
    print(k, json.dumps(r), flush=True)
