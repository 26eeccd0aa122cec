"""Small fixed workload for ncu captures (not part of the product)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_08417_b200 import engine, inputs, workloads, _lib
which = sys.argv[1] if len(sys.argv) > 1 else "c5s"
eng = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if which == "c5s":
    cfgs = [workloads.c5(seed=s, horizon_s=60.0) for s in range(1, 9)]
elif which == "c5":
    cfgs = workloads.c5_sweep(seeds=range(1, 65))
elif which == "c5h120":
    import dataclasses
    cfgs = [dataclasses.replace(c, horizon_s=120.0) for c in workloads.c5_sweep(seeds=range(1, 65))]
else:
    cfgs = [workloads.c2(seed=s) for s in range(1, 65)]
inp = inputs.build_inputs(cfgs, engine=eng, mode=_lib.MODE_HISTOGRAM)
db = engine.DeviceBatch(inp)
db.launch(); torch.cuda.synchronize()
db.launch(); torch.cuda.synchronize()
print("requests", db.fetch().total_requests)
