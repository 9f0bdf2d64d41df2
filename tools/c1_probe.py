import sys, json, os
sys.path.insert(0, '.')
import bench
r = bench.c1_leg(1)
print(os.environ.get("GPCX_TCP_BUF"), json.dumps({"c1_ms": r["ms_per_request"]}))
