"""Config-4 tail probe (not part of the product): each client-count class of the
2,688-scenario sweep (6 variants x 64 seeds = 384 scenarios) timed alone, with
the windowed engine's per-phase cycle split, then the whole sweep.

    python tools/c4_probe.py [--nw 1|2|auto]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_08417_b200 import _lib, engine, inputs, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--nw", default="auto")
ap.add_argument("--classes", default="10,30,100,300,1000,3000,10000")
args = ap.parse_args()
if args.nw != "auto":
    os.environ["OTF_WIN_NW"] = args.nw


def run(cfgs, name):
    inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM, pin=True)
    db = engine.DeviceBatch(inp, pin=True)
    db.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    br = db.fetch()
    st = br.stats.sum(0).astype(float)
    win = max(1.0, st[_lib.ST["windows"]])
    tot = max(1.0, st[_lib.ST["cyc_total"]])
    per = br.stats[:, _lib.ST["cyc_total"]].astype(float)
    print(json.dumps(dict(name=name, scenarios=len(cfgs), ms=round(ms, 2), requests=int(br.total_requests),
                          req_per_s=br.total_requests / (ms / 1e3), windows_per_scn=win / len(cfgs),
                          cycles_per_window=tot / win,
                          split={k: round(st[_lib.ST[k]] / tot, 3) for k in ("cyc_scan", "cyc_sort", "cyc_server",
                                                                              "cyc_clients")},
                          scn_cycles_max=per.max(), scn_cycles_mean=per.mean(),
                          status_max=int(br.status.max()))), flush=True)


for n in [int(x) for x in args.classes.split(",")]:
    run([workloads.c4(seed=s, clients=n, variant=v) for v in workloads.C4_VARIANTS for s in range(1, 65)], f"c4_N{n}")
run(workloads.c4_sweep(), "c4_full")

# per launch group of the full sweep: when each group's kernels start and end (events on
# each group's stream), and the longest scenario of each group
cfgs = workloads.c4_sweep()
inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM, pin=True)
db = engine.DeviceBatch(inp, pin=True)
db.launch()
torch.cuda.synchronize()
import ctypes
s = torch.cuda.current_stream()
t_origin = torch.cuda.Event(enable_timing=True)
db.generate(s)
t_origin.record(s)
evs = []
streams = [s] + db.streams
for gb, st in zip(db.groups, streams):
    if st is not s:
        st.wait_event(t_origin)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    _lib.check(db.lib.otf_run_batch(ctypes.byref(gb), inp.engine, st.cuda_stream), "run")
    b.record(st)
    evs.append((a, b, gb))
torch.cuda.synchronize()
br = db.fetch()
order = db.order.cpu().numpy()
off = 0
for a, b, gb in evs:
    k = gb.n_scenarios
    first = (gb.order - db.order.data_ptr()) // 4
    idx = order[first:first + k]
    cyc = br.stats[idx, _lib.ST["cyc_total"]].astype(float)
    ncl = sorted({cfgs[i].clients for i in idx})
    print(json.dumps(dict(group_scenarios=k, clients=ncl, smem=gb.shared_bytes, start_ms=round(t_origin.elapsed_time(a), 1),
                          end_ms=round(t_origin.elapsed_time(b), 1), max_scn_ms=round(cyc.max() / 1965e3, 1))), flush=True)
