"""Small windowed- and exact-engine batch for compute-sanitizer (not part of the product).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
Runs generation + both engines + the summary pass in both modes on a few
small scenarios (two warps and one warp per scenario) and checks them against
the oracle, so a sanitizer run also proves the sanitized launches computed the
right thing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle
from paper_2603_08417_b200 import engine, workloads
from tests import parity

cfgs = [workloads.c1(seed=1), workloads.c2(seed=2, horizon_s=40.0), workloads.c3(seed=3, fraction=0.1, horizon_s=40.0),
        workloads.c5(seed=4, clients=120, horizon_s=30.0)]
for nw in ("1", "2", "3"):
    os.environ["OTF_WIN_NW"] = nw
    for eng in ("windowed", "exact"):
        for mode in ("records", "histogram"):
            res = engine.run_batch(cfgs, mode=mode, engine=eng)
            if mode == "records":
                for c, r in zip(cfgs, res):
                    errs = parity.compare(r.arrays, oracle.run(c))
                    assert not errs, errs[:5]
            print(f"nw={nw} {eng} {mode}: ok", flush=True)
