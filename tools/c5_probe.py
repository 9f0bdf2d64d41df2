"""Why is C5 slower inside the full bench than alone?  Runs the C5 leg
after different preceding legs in one process (diagnostic, not product)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


def c5(tag):
    r = bench.c5_leg(1)
    print(tag, json.dumps({k: round(r[k], 2) for k in ("chains_per_s", "seconds")}), flush=True)


order = sys.argv[1:]
for step in order:
    if step == "c5":
        c5("c5")
    elif step == "c4":
        bench.matmul_c4_leg(bench.Dist(1), 3, 1)
        print("c4 done", flush=True)
    elif step == "c2":
        bench.matmul_device_leg(5, 2)
        print("c2 done", flush=True)
    elif step == "lut":
        bench.lut_device_leg(bench.Dist(1), 10, 3, 0)
        print("lut done", flush=True)
    elif step == "sleep":
        time.sleep(5)
