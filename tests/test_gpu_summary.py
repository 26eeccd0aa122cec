"""GPU: the fused QoE block and the histogram-mode summary, field by field.

* every golden fixture, both engines, both modes: the device's otf_qoe equals
  the block restated from the reference's own records (oracle.qoe_block), and
  summary() in histogram mode equals the summary the reference wrote;
* the benchmark workloads in full -- all 1,024 config-5 and all 2,688 config-4
  scenarios in histogram mode -- against the C oracle run in a process pool:
  every histogram bin and counter, the backend stats, and the summary
  statistics (order statistics, registration-order stall sum, exact sums)
  bit for bit;
* a stratified records-mode sample (every config-4 client count incl. 10,000,
  every variant, and config-5 points) bit-exact against the oracle's records.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2603_08417_b200 import _lib, engine, workloads
from paper_2603_08417_b200.config import ExperimentConfig
from tests import parity

pytestmark = pytest.mark.gpu

QOE_INT = ("lat_hist", "path_count", "stall_hist", "rank_count", "n_requests", "n_sessions", "n_segments",
           "n_finished", "n_started", "n_stalls", "n_lat_tail", "n_stall_tail")
QOE_FLOAT = ("latency_sum", "stall_time_sum", "startup_delay_sum", "latency_p50", "latency_p99")


def _cfg(meta):
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    cfg.zipf_exponent = meta["zipf_exponent"]
    return cfg


def qoe_errors(got: dict, want: dict, tag) -> list[str]:
    errs = []
    for k in QOE_INT:
        g = got[k][:len(want[k])] if isinstance(want[k], list) else got[k]
        if g != want[k]:
            errs.append(f"{tag} {k}: {g} != {want[k]}")
    for k in QOE_FLOAT:                                 # bit-exact (north star: <= 1e-6 relative)
        if np.float64(got[k]).view(np.int64) != np.float64(want[k]).view(np.int64):
            errs.append(f"{tag} {k}: {got[k]!r} != {want[k]!r}")
    if not got["summary_flags"] & _lib.Q_ORDER_STATS:
        errs.append(f"{tag}: summary pass did not run (flags {got['summary_flags']:#x})")
    return errs


def _pool_map(fn, items):
    ctx = mp.get_context("fork")
    with ctx.Pool(os.cpu_count() or 1) as pool:
        return pool.map(fn, items, chunksize=1)


@pytest.fixture(scope="module")
def golden():
    return {n: parity.load_golden(n) for n in parity.golden_names()}


@pytest.mark.parametrize("eng", ["exact", "windowed"])
@pytest.mark.parametrize("mode", ["histogram", "records"])
def test_qoe_blocks_and_summaries_vs_reference(golden, eng, mode):
    names = sorted(golden)
    results = engine.run_batch([_cfg(golden[n][1]) for n in names], mode=mode, engine=eng)
    errs = []
    for n, res in zip(names, results):
        want_arrays, meta = golden[n]
        errs += qoe_errors(res.qoe, oracle.qoe_block(want_arrays), n)
        if mode == "histogram":
            got, want = res.summary(), dict(meta["summary"])
            if meta["popularity"] != "uniform":
                got.pop("fingerprint"), want.pop("fingerprint")
            if got != want:
                errs.append(f"{n} summary: {got} != {want}")
    assert not errs, "\n".join(errs[:20])


def _full_sweep_vs_oracle(cfgs):
    ctx = mp.get_context("fork")
    with ctx.Pool(os.cpu_count() or 1) as pool:        # the CPU oracle runs while the GPU does
        pending = pool.map_async(oracle.run_qoe, cfgs, chunksize=1)
        hist = engine.run_batch(cfgs, mode="histogram")
        want = pending.get()
    errs, fallbacks = [], 0
    for i, (h, w) in enumerate(zip(hist, want)):
        fallbacks += h.engine != "windowed"
        errs += qoe_errors(h.qoe, w, f"scenario {i} ({cfgs[i].variant}, seed {cfgs[i].seed}, N={cfgs[i].clients})")
        if list(h.stats_raw[:18]) != w["stats"]:
            errs.append(f"scenario {i} stats: {list(h.stats_raw[:18])} != {w['stats']}")
        if int(h.counts[3]) != w["n_job"]:
            errs.append(f"scenario {i} jobs: {h.counts[3]} != {w['n_job']}")
    return hist, errs, fallbacks


def test_config5_full_sweep_every_scenario_vs_oracle():
    """All 1,024 benchmark scenarios (2,800 clients, 600 s, 10-rank ladder)."""
    cfgs = workloads.c5_sweep()
    hist, errs, fallbacks = _full_sweep_vs_oracle(cfgs)
    assert not errs, f"{len(errs)} mismatches:\n" + "\n".join(errs[:20])
    assert fallbacks == 0
    assert sum(h.qoe["n_requests"] for h in hist) > 1_500_000_000


def test_config4_full_sweep_every_scenario_vs_oracle():
    """All 2,688 config-4 scenarios (10..10,000 clients x 6 variants x 64 seeds)."""
    cfgs = workloads.c4_sweep()
    hist, errs, _ = _full_sweep_vs_oracle(cfgs)
    assert not errs, f"{len(errs)} mismatches:\n" + "\n".join(errs[:20])


def _stratified():
    cfgs = []
    for k, n in enumerate(workloads.C4_CLIENTS):        # every client count, every variant across them
        for j in range(4):
            v = workloads.C4_VARIANTS[(k + j) % len(workloads.C4_VARIANTS)]
            cfgs.append(workloads.c4(seed=11 + 4 * k + j, clients=n, variant=v))
    for s, v, f in ((21, "TC", 0.05), (22, "TCP", 0.10), (23, "TCF", 0.20), (24, "TCPF", 0.50)):
        cfgs.append(workloads.c5(seed=s, variant=v, fraction=f))
    return cfgs


def test_records_stratified_sample_bit_exact():
    """32 scenarios in records mode, every record field bit-exact vs the oracle."""
    cfgs = _stratified()
    assert len(cfgs) == 32 and any(c.clients == 10000 for c in cfgs) and any(c.variant == "TCF" for c in cfgs)
    ctx = mp.get_context("fork")
    with ctx.Pool(os.cpu_count() or 1) as pool:
        pending = pool.map_async(oracle.run, cfgs, chunksize=1)
        got = engine.run_batch(cfgs, mode="records")
        want = pending.get()
    for cfg, res, ref in zip(cfgs, got, want):
        errs = parity.compare(res.arrays, ref)
        assert not errs, (cfg.variant, cfg.clients, cfg.seed, errs[:5])
        errs = parity.compare_stats(res.backend_stats, oracle.backend_stats(ref, "C" in cfg.variant))
        assert not errs, errs
        assert not qoe_errors(res.qoe, oracle.qoe_block(ref), cfg.seed)


def test_tail_overflow_rerun_is_exact(golden):
    """Summary tails far too small: the scenarios are re-run with the exact counts."""
    names = ["c1_seed1", "grid_c24_k4_t2_TCP", "c3_f05_h90"]
    cfgs = [_cfg(golden[n][1]) for n in names]
    for caps in ((2, 1, 1, 1), (1 << 20, 1 << 20, 1, 1 << 20)):   # engine tails / the summary's gather
        res = engine.run_batch(cfgs, mode="histogram", _tail_caps=[caps] * len(cfgs))
        for n, r in zip(names, res):
            want = oracle.qoe_block(golden[n][0])
            assert r.attempts == (2 if caps[0] == 2 or want["n_stall_tail"] > 1 else 1), (n, caps, r.attempts)
            assert not qoe_errors(r.qoe, want, n)


def test_histogram_summary_exact_engine_matches_windowed():
    cfgs = [workloads.c2(seed=s) for s in (1, 2)] + [workloads.c3(seed=3, fraction=0.0)]
    a = engine.run_batch(cfgs, mode="histogram", engine="exact")
    b = engine.run_batch(cfgs, mode="histogram", engine="windowed")
    for x, y in zip(a, b):
        assert x.summary() == y.summary()
        assert not qoe_errors(x.qoe, y.qoe, "exact-vs-windowed")


def test_records_only_views_raise_in_histogram_mode():
    r = engine.run_batch([workloads.c1(seed=2)], mode="histogram")[0]
    assert r.summary()["requests"] > 0
    with pytest.raises(_lib.OtfError):
        r.requests


def test_list_overflow_reruns_windowed_with_larger_list():
    """A transcode-bound config-5 point (TCP, cache 0.5% of the ladder, seed 60) sees a
    burst of more simultaneous requests than the default 256-entry window list: the
    engine flags OTF_S_LIST_OVERFLOW and run_batch re-runs it on the windowed engine
    with a 4x list (not the one-thread exact engine), bit-exact vs the oracle."""
    cfg = workloads.c5(seed=60, variant="TCP", fraction=0.005)
    res = engine.run_batch([cfg], mode="histogram")[0]
    assert res.engine == "windowed" and res.list_cap >= 1024, (res.engine, res.list_cap)
    want = oracle.run_qoe(cfg)
    errs = qoe_errors(res.qoe, want, "c5t seed 60")
    assert not errs, errs
    assert list(res.stats_raw[:18]) == want["stats"]


def test_run_to_run_bit_identical():
    """Two launches of the same batch produce identical QoE blocks, stats and counts,
    bit for bit (the float sums are exact / registration-ordered, not atomic-order
    dependent), in every kernel shape."""
    import os
    cfgs = [workloads.c5(seed=s, variant=v, clients=600, horizon_s=120.0) for s in (1, 2) for v in ("TC", "TCPF")]
    for nw in ("1", "2", "3"):
        os.environ["OTF_WIN_NW"] = nw
        try:
            a = engine.run_batch(cfgs, mode="histogram")
            b = engine.run_batch(cfgs, mode="histogram")
        finally:
            os.environ.pop("OTF_WIN_NW", None)
        for x, y in zip(a, b):
            # stats slots after OTF_ST_WINDOWS (22) are cycle counters: timing, not results
            assert np.array_equal(x.qoe_row, y.qoe_row) and np.array_equal(x.stats_raw[:23], y.stats_raw[:23])
            assert np.array_equal(x.counts, y.counts)
