"""Timing probe for engine calibration (not part of the product)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_2603_08417_b200 import engine, inputs, workloads, _lib

def timeit(name, cfgs, eng, reps=2):
    t0 = time.time()
    inp = inputs.build_inputs(cfgs, engine=eng, mode=_lib.MODE_HISTOGRAM)
    t1 = time.time()
    db = engine.DeviceBatch(inp)
    db.launch(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); db.launch(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    br = db.fetch()
    req = br.total_requests
    if eng == 1:
        st = br.stats.sum(0)
        tot = max(1, st[27])
        print("  windows/scn", st[22] / len(cfgs), "cycles/window", tot / max(1, st[22]),
              "scan %.2f sort %.2f server %.2f clients %.2f" % (st[23]/tot, st[24]/tot, st[25]/tot, st[26]/tot),
              "pops/scn", st[20]/len(cfgs), "ready", st[21]/len(cfgs),
              "| local(concurrent) %.2f | parallel server windows %.3f" % (st[28]/tot, st[29] / max(1, st[22])))
        if os.environ.get("OTF_DIAG"):
            for name, rows in (("all", slice(None)), ("TCP", [i for i in range(len(cfgs)) if i % 16 in (4, 5, 6, 7)])):
                S = br.stats[rows].sum(0).astype(float)
                print("  diag[%s]: per window: server %.0f requests %.0f workers %.0f handoffs %.0f clients %.0f local %.0f "
                      "scan %.0f sort %.0f cycles; requests/window %.1f" % (name,
                      S[25] / S[22], S[29] / S[22], S[30] / S[22], S[31] / S[22], S[26] / S[22], S[28] / S[22],
                      S[23] / S[22], S[24] / S[22], br.counts[rows, 0].sum() / S[22]))
        if os.environ.get("OTF_FAR_DIAG"):
            v = br.stats[:, 28].astype(np.int64)
            print("  far-diag: far pushes per scenario %.1f (of which beyond the horizon %.1f), windows %.0f" % (
                (v & 0xffffffff).sum() / len(cfgs), (v >> 32).sum() / len(cfgs), st[22] / len(cfgs)))
        if os.environ.get("OTF_PAR_DIAG"):
            print("  par-diag: per window: parallel_ok %.0f, group replay %.0f, prefix+effects+handoffs %.0f, server total %.0f" % (
                st[30] / st[22], st[28] / st[22], st[31] / st[22], st[25] / st[22]))
        per = br.stats[:, 27].astype(float)
        print("  scenario cycles: mean %.3g max %.3g (max/mean %.3f), max at %d" % (per.mean(), per.max(), per.max() / per.mean(), per.argmax()))
        if len(cfgs) % 16 == 0:
            g = per.reshape(-1, 16).mean(0)
            print("  by (variant, fraction) slot:", " ".join("%.3g" % x for x in g))
    print(json.dumps(dict(name=name, engine=eng, scenarios=len(cfgs), build_s=round(t1-t0,2), ms=round(best,2),
                          requests=req, req_per_s=req/(best/1e3), status=int(br.status.max()))), flush=True)

which = sys.argv[1:] or ["c1", "c2", "c5s"]
for w in which:
    if w == "c1": timeit("c1x64", [workloads.c1(seed=s) for s in range(1, 65)], 0)
    if w == "c2": timeit("c2x64", [workloads.c2(seed=s) for s in range(1, 65)], 0)
    if w == "c2w": timeit("c2x64", [workloads.c2(seed=s) for s in range(1, 65)], 1)
    if w == "c5s": timeit("c5x8_h60", [workloads.c5(seed=s, horizon_s=60.0) for s in range(1, 9)], 0, reps=1)
    if w == "c5": timeit("c5x64", workloads.c5_sweep(seeds=range(1, 5)), 0, reps=1)
for w in which:
    if w == "c1w": timeit("c1x64", [workloads.c1(seed=s) for s in range(1, 65)], 1)
    if w == "c5sw": timeit("c5x8_h60", [workloads.c5(seed=s, horizon_s=60.0) for s in range(1, 9)], 1, reps=1)
    if w == "c5w": timeit("c5x64", workloads.c5_sweep(seeds=range(1, 5)), 1, reps=1)
    if w == "c5fw": timeit("c5x1024", workloads.c5_sweep(seeds=range(1, 65)), 1, reps=1)
    if w == "c5tw": timeit("c5t_x1024", workloads.c5t_sweep(seeds=range(1, 65)), 1, reps=1)
for w in which:
    if w == "c4w":
        cfgs = workloads.c4_sweep(seeds=range(1, 9))
        timeit("c4x8seeds", cfgs, 1, reps=1)
    if w == "c4T10k":
        timeit("c4_10k_T", [workloads.c4(seed=s, clients=10000, variant=v) for s in range(1, 9)
                             for v in ("T", "TC")], 1, reps=1)
    if w == "c4big":
        cfgs = [workloads.c4(seed=s, clients=10000, variant=v) for s in (1, 2) for v in ("TC", "TCPF")]
        timeit("c4_10k", cfgs, 1, reps=1)
