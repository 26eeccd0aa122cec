"""Strong-scaling probe (not part of the product): the per-rank shard of the
1,024-scenario config-5 sweep at N = 1, 2, 4, 8 GPUs, each run on this one GPU.

Rank r of an N-GPU strong-scaling run owns 64/N seed groups (dist.shard), i.e.
1,024/N scenarios, and its time is what bounds the N-GPU step (the ranks run
concurrently and the only collective is the ~1 MB gather).  So the N-GPU
throughput is predicted as 1,024-scenario requests / max shard time; the
shards are equal-cost (every seed group has the same 16 variants x cache
points), so one shard is timed per N.

    python tools/strong_probe.py [--nw 1|2|auto] [--ns 1,2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_08417_b200 import _lib, dist, engine, inputs, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--nw", default="auto")
ap.add_argument("--ns", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--seeds", type=int, default=0, help="time the first SEEDS seed groups instead of the N-GPU shards")
args = ap.parse_args()
if args.nw != "auto":
    os.environ["OTF_WIN_NW"] = args.nw
full = workloads.c5_sweep(seeds=range(1, 65))
for n in ([1] if args.seeds else [int(x) for x in args.ns.split(",")]):
    mine = dist.shard(full, 0, n)
    cfgs = [full[i] for i in mine] if not args.seeds else full[:16 * args.seeds]
    inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM, pin=True)
    db = engine.DeviceBatch(inp, pin=True)
    db.launch()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        db.launch()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    br = db.fetch()
    req = br.total_requests
    print(json.dumps(dict(n_gpus=n, nw=args.nw, scenarios=len(cfgs), shard_ms=round(best, 2), shard_requests=req,
                          predicted_total_req_per_s=req * n / (best / 1e3),
                          status_max=int(br.status.max()))), flush=True)
