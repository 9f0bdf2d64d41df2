"""A/B of the C5 leg between two checkouts on the same box (bench.c5_leg
imported from each tree in a fresh process):  python tools/c5_ab.py DIR"""
import json
import sys

sys.path.insert(0, sys.argv[1])
import bench  # noqa: E402

r = bench.c5_leg(1)
print(json.dumps({"tree": sys.argv[1], "chains_per_s": round(r["chains_per_s"], 2),
                  "phases": r["phases_ms_per_request"]}), flush=True)
