"""GPU parity: libotfgpu.so vs the reference's golden outputs and the C oracle.

Every test calls through the C ABI (paper_2603_08417_b200 -> ctypes ->
libotfgpu.so).  Discrete fields must match exactly; float fields are compared
bit-for-bit (the engine keeps the reference's operation order with FMA
contraction disabled) -- the north star's bar is <= 1e-6 relative, bit-exact
is what is asserted.
"""

import numpy as np
import pytest

from oracle import oracle
from paper_2603_08417_b200 import _lib, engine, inputs, workloads
from paper_2603_08417_b200.config import ExperimentConfig
from tests import parity

pytestmark = pytest.mark.gpu


def _cfg(meta):
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    cfg.zipf_exponent = meta["zipf_exponent"]
    return cfg


def _assert_parity(res, want, stats_want=None):
    errs = parity.compare(res.arrays, want)
    assert not errs, "\n".join(errs[:20])
    if stats_want is not None:
        errs = parity.compare_stats(res.backend_stats, stats_want)
        assert not errs, "\n".join(errs)


@pytest.fixture(scope="module")
def golden():
    return {n: parity.load_golden(n) for n in parity.golden_names()}


def test_size_tables_match_oracle(golden):
    cfgs = [_cfg(m) for _, m in golden.values()]
    inp = inputs.build_inputs(cfgs, mode=_lib.MODE_HISTOGRAM, engine=_lib.ENGINE_EXACT)
    db = engine.DeviceBatch(inp)
    db.launch()
    br = db.fetch()
    for i, cfg in enumerate(cfgs):
        want, _ = oracle.Prepared(cfg).sizes()
        assert np.array_equal(br.sizes(i), want), cfg


@pytest.mark.parametrize("eng,nw", [("exact", ""), ("windowed", ""), ("windowed", "1"), ("windowed", "2"),
                                    ("windowed", "3")])
def test_golden_parity_batched(golden, eng, nw, monkeypatch):
    """All golden configs in ONE launch, each bit-exact vs the reference; the windowed
    engine also with each kernel shape forced (1: one warp, 2: two warps with the
    256-register budget, 3: two warps with the 128-register budget of 7 per SM)."""
    if nw:
        monkeypatch.setenv("OTF_WIN_NW", nw)
    names = sorted(golden)
    cfgs = [_cfg(golden[n][1]) for n in names]
    results = engine.run_batch(cfgs, mode="records", engine=eng)
    for n, res in zip(names, results):
        want, meta = golden[n]
        _assert_parity(res, want, meta["backend_stats"])


def test_summary_matches_reference(golden):
    names = ["c1_seed1", "grid_c24_k4_t2_TCPF", "c3_f05_h90"]
    results = engine.run_batch([_cfg(golden[n][1]) for n in names], mode="records")
    for n, res in zip(names, results):
        want = golden[n][1]["summary"]
        got = res.summary()
        for k in ("requests", "sessions", "jobs", "instant_fraction", "latency_p50_s", "latency_p99_s",
                  "stalls_mean", "stall_time_total_s", "mean_rank", "quality_fractions", "variant"):
            assert got.get(k) == want.get(k), (n, k, got.get(k), want.get(k))


def test_run_experiment_dropin_objects(golden):
    want, meta = golden["grid_c24_k4_t2_TCP"]
    res = engine.run_experiment(_cfg(meta))
    assert len(res.requests) == len(want["req_id"])
    r0 = res.requests[0]
    assert r0.path in ("storage", "cache", "waited_inflight", "transcoded")
    assert res.jobs[0].origin in ("demand", "speculative")
    assert sum(len(s.segments) for s in res.sessions) == len(want["seg_index"])


def _oracle_cmp(cfgs, eng="windowed"):
    results = engine.run_batch(cfgs, mode="records", engine=eng)
    for cfg, res in zip(cfgs, results):
        ref = oracle.run(cfg)
        errs = parity.compare(res.arrays, ref)
        assert not errs, (cfg, errs[:10])
        errs = parity.compare_stats(res.backend_stats, oracle.backend_stats(ref, "C" in cfg.variant))
        assert not errs, errs
    return results


def test_config2_full_horizon_vs_oracle():
    """BASELINE config 2 at full size (100 clients, 600 s) over several seeds."""
    _oracle_cmp([workloads.c2(seed=s) for s in (1, 2, 3)])


def test_config3_cache_sweep_vs_oracle():
    """BASELINE config 3: cache fraction 0..1 in 0.1 steps (one launch)."""
    _oracle_cmp([workloads.c3(seed=5, fraction=f / 10) for f in range(11)])


def test_config1_seeds_vs_oracle():
    _oracle_cmp([workloads.c1(seed=s) for s in range(1, 9)])


def test_config4_points_vs_oracle():
    """BASELINE config 4 sample points (client-count sweep x variants)."""
    cfgs = [workloads.c4(seed=s, clients=n, variant=v)
            for (s, n, v) in [(1, 10, "B"), (2, 30, "T"), (3, 100, "TC"), (4, 300, "TCP"), (5, 30, "TCF"),
                              (6, 100, "TCPF")]]
    _oracle_cmp(cfgs)


def test_config4_largest_points_vs_oracle():
    """BASELINE config 4 at its largest client counts, full 600 s horizon: 10,000 clients
    (windows of ~180 requests: the shared-memory bitonic sort, the parallel server pass
    at up to 256 requests, the largest shared-memory class) and 3,000 clients."""
    _oracle_cmp([workloads.c4(seed=7, clients=10000, variant="TCP"),
                 workloads.c4(seed=8, clients=3000, variant="TCPF")])


def test_config5_point_vs_oracle():
    """BASELINE config 5 (10-rank ladder) at reduced client count and horizon."""
    _oracle_cmp([workloads.c5(seed=s, clients=400, horizon_s=120.0, variant=v)
                 for s, v in [(1, "TCPF"), (2, "TCP")]])


def test_windowed_large_catalogs_vs_oracle():
    """Catalogs past round 1's limits stay on the windowed engine: 40,000 descriptors
    (50 sequences x 80 s at 1 s segments x the 10-rank ladder: 16-bit unsigned
    descriptor ids) and 100 sequences (the catalog tables read from global memory)."""
    from paper_2603_08417_b200.workloads import _seqs
    big = workloads.c5(seed=3, clients=300, horizon_s=150.0, variant="TCP", sequences=_seqs(50, duration=80.0),
                       sequence_duration_s=80.0)
    wide = workloads.c2(seed=4, clients=200, horizon_s=200.0, variant="TCPF", sequences=_seqs(100))
    results = _oracle_cmp([big, wide])
    assert [r.engine for r in results] == ["windowed", "windowed"]
    from paper_2603_08417_b200 import inputs as _inp
    low = _inp.lower(big)
    assert len(low.seq_ids) * low.n_ranks * max(low.counts) == 40_000


def test_histogram_mode_matches_records():
    cfgs = [workloads.c3(seed=7, fraction=f) for f in (0.0, 0.3, 1.0)] + [workloads.c1(seed=3)]
    rec = engine.run_batch(cfgs, mode="records")
    hist = engine.run_batch(cfgs, mode="histogram")
    for r, h in zip(rec, hist):
        a = r.arrays
        q = h.qoe
        assert q["n_requests"] == len(a["req_id"])
        assert q["n_sessions"] == len(a["sess_client"])
        assert q["n_segments"] == len(a["seg_index"])
        assert q["path_count"] == [int((a["req_path"] == p).sum()) for p in range(5)]
        lat = a["req_response"] - a["req_arrival"]
        assert q["lat_hist"][0] == int((lat < 0.010).sum())
        assert sum(q["lat_hist"]) == len(lat)
        ranks = np.bincount(a["seg_rep"], minlength=_lib.RANK_BINS)[:_lib.RANK_BINS]
        assert q["rank_count"] == list(ranks)
        stalls = np.minimum(a["sess_stalls"], 31)
        assert q["stall_hist"] == list(np.bincount(stalls, minlength=32))
        assert q["stall_time_sum"] == pytest.approx(float(a["sess_stall_time"].sum()), rel=1e-9, abs=1e-9)
        assert np.array_equal(r.stats_raw[:18], h.stats_raw[:18])


def test_records_mode_chunks_to_fit_device_memory(monkeypatch):
    """A records-mode sweep whose record buffers exceed half the free device memory
    runs in chunks; the results equal the one-launch run."""
    import torch
    cfgs = [workloads.c3(seed=4, fraction=f) for f in (0.0, 0.2, 0.6)] + [workloads.c1(seed=6)]
    whole = engine.run_batch(cfgs, mode="records")
    free, total = torch.cuda.mem_get_info()
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda *a, **k: (60_000_000, total))   # ~1 config per chunk
    chunked = engine.run_batch(cfgs, mode="records")
    for a, b in zip(whole, chunked):
        errs = parity.compare(b.arrays, a.arrays)
        assert not errs, errs[:5]


def test_no_cpu_fallback_without_library(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libotfgpu.so")
    with pytest.raises(_lib.OtfError):
        engine.run_experiment(workloads.c1())


def test_fallback_and_retry_paths(golden):
    """Windowed engine hands zero-latency scenarios to the exact engine; record and
    noise-table overflows are re-run with exact sizes -- results stay bit-exact."""
    want, meta = golden["edge_latency0"]
    res = engine.run_batch([_cfg(meta)], mode="records", engine="windowed")[0]
    assert res.engine == "exact"
    _assert_parity(res, want, meta["backend_stats"])
    want, meta = golden["grid_c24_k4_t2_TCP"]
    res = engine.run_batch([_cfg(meta)], mode="records", _caps=[(10, 3, 10, 5)])[0]
    assert res.attempts == 2 and res.engine == "windowed"
    _assert_parity(res, want, meta["backend_stats"])
    res = engine.run_batch([_cfg(meta)], mode="records", _eps_scale=0.02)[0]
    assert res.attempts >= 2
    _assert_parity(res, want, meta["backend_stats"])


def test_run_sharded_single_rank():
    from paper_2603_08417_b200 import dist as odist
    cfgs = [workloads.c1(seed=s) for s in range(1, 5)]
    blocks = odist.run_sharded(cfgs)
    ref = engine.run_batch(cfgs, mode="histogram")
    assert [int(b[0]) for b in blocks] == [0, 1, 2, 3]
    assert [int(b[1]) for b in blocks] == [r.status for r in ref]
    assert [int(b[2]) for b in blocks] == [r.qoe["n_requests"] for r in ref]


def test_cli_matrix_matches_reference_bundles(tmp_path):
    """`matrix` (72 configs, one launch) writes the reference's bundle for a grid point."""
    import filecmp
    import os
    from paper_2603_08417_b200 import cli
    assert cli.main(["run", "--variant", "T", "--clients", "4", "--seed", "1", "--out", str(tmp_path / "run")]) == 0
    assert (tmp_path / "run" / "requests.csv").exists()
    assert cli.main(["matrix", "--out", str(tmp_path / "m")]) == 0
    assert len(os.listdir(tmp_path / "m")) == 72
    ref_dir = os.path.join(parity.GOLDEN_DIR, "csv_matrix")
    for name in sorted(os.listdir(ref_dir)):            # byte-identical to the reference's own bundle
        for f in ("requests.csv", "sessions.csv", "segments.csv", "jobs.csv", "config.json", "summary.json"):
            assert filecmp.cmp(tmp_path / "m" / name / f, os.path.join(ref_dir, name, f), shallow=False), (name, f)
