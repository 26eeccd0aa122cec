"""Time the pieces of engine.run_batch on config 5 (not part of the product)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_08417_b200 import engine, inputs, workloads, _lib
cfgs = workloads.c5_sweep()
engine.run_batch(cfgs[:16], mode="histograms")          # warm up CUDA / pinned allocator
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lows = [inputs.lower(inputs.ExperimentConfig.from_reference(c)) for c in cfgs]
    t1 = time.perf_counter()
    inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM, pin=True)
    t2 = time.perf_counter()
    db = engine.DeviceBatch(inp, pin=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    db.launch()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    br = db.fetch()
    res = [br.result(k) for k in range(len(cfgs))]
    t5 = time.perf_counter()
    a = time.perf_counter()
    engine.run_batch(cfgs, mode="histograms")
    torch.cuda.synchronize()
    b = time.perf_counter()
    print(f"lower {t1-t0:.3f}  build_inputs {t2-t1:.3f}  DeviceBatch(H2D) {t3-t2:.3f}  kernel {t4-t3:.3f}  fetch+results {t5-t4:.3f}  | run_batch {b-a:.3f}  cores {os.cpu_count()}", flush=True)
