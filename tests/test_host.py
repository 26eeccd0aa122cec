"""CPU-side tests: the C ABI loads and exports its symbols, the host input
builder reproduces the reference's input streams, config parity."""

import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from oracle import oracle
from paper_2603_08417_b200 import _lib, inputs, workloads
from paper_2603_08417_b200.config import ConfigError, ExperimentConfig, scenario_matrix
from tests import parity

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    header = open(os.path.join(ROOT, "include", "otfgpu.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|int32_t|double|size_t|const char \*)\s*\*?\s*(otf_\w+)\s*\(",
                              header, re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.otf_version() == _lib.ABI_VERSION


def test_struct_layouts_match_c():
    L = _lib.lib()
    assert L.otf_sizeof_scenario() == ctypes.sizeof(_lib.Scenario)
    assert L.otf_sizeof_batch() == ctypes.sizeof(_lib.Batch)
    assert L.otf_sizeof_qoe() == ctypes.sizeof(_lib.Qoe)


def test_run_batch_rejects_bad_arguments():
    L = _lib.lib()
    b = _lib.Batch()
    b.n_scenarios = 1
    rc = L.otf_run_batch(ctypes.byref(b), 0, None)
    assert rc == 1
    assert b"missing device buffer" in L.otf_last_error()
    assert L.otf_run_batch(None, 0, None) == 1


def test_scratch_bytes_positive():
    L = _lib.lib()
    for eng in (0, 1):
        assert L.otf_scratch_bytes(eng, 100, 4, 50, 5, 10) > 100 * 64
        assert L.otf_shared_bytes(1, 100, 4, 50, 5, 10) < 48 * 1024
        assert L.otf_shared_bytes(0, 100, 4, 50, 5, 10) == 0


def full_pool(inp) -> np.ndarray:
    """The whole f64 pool as the device builds it: the device-generated prefix
    replayed by the host generators (inputs.host_generate), then the host part."""
    return np.concatenate([inputs.host_generate(inp), inp.f64])


@pytest.mark.parametrize("name", ["c1_seed1", "c2_seed1_h120", "edge_partial_seg"])
def test_traces_match_oracle(name):
    """otf_build_traces (C++, glibc exp, 3.12 sum) == oracle traces (which match the reference)."""
    _, meta = parity.load_golden(name)
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    inp = inputs.build_inputs([cfg], mode=_lib.MODE_HISTOGRAM)
    sc = inp.scenarios[0]
    prep = oracle.Prepared(cfg)
    starts, values, pbits, period = prep.traces()
    n = sc.n_samples
    pool = full_pool(inp)
    got_vals = pool[sc.off_values:sc.off_values + cfg.clients * n].reshape(cfg.clients, n)
    got_pbits = pool[sc.off_pbits:sc.off_pbits + cfg.clients]
    assert sc.period == period
    assert np.array_equal(pool[sc.off_starts:sc.off_starts + n], starts)
    assert np.array_equal(got_vals.view(np.int64), values.view(np.int64))
    assert np.array_equal(got_pbits.view(np.int64), pbits.view(np.int64))


def test_traces_match_reference_semantics():
    """Spot-check a trace against a pure-Python restatement of synthetic_trace."""
    cfg = ExperimentConfig(seed=42, clients=3)
    inp = inputs.build_inputs([cfg], mode=_lib.MODE_HISTOGRAM)
    sc = inp.scenarios[0]
    n = sc.n_samples
    pool = full_pool(inp)
    for c in range(3):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([42, 2, c])))
        mu = math.log(17e6)
        decay = math.exp(-0.08)
        spread = 0.35 * math.sqrt(1.0 - decay * decay)
        x = mu + 0.35 * rng.standard_normal()
        vals = []
        t = 0.0
        while t < 600.0:
            vals.append(min(max(math.exp(x), 2e6), 400e6))
            x = mu + (x - mu) * decay + spread * rng.standard_normal()
            t += 1.0
        got = pool[sc.off_values + c * n: sc.off_values + (c + 1) * n]
        assert list(got) == vals
        pb = sum(v * 1.0 for v in vals)
        assert pool[sc.off_pbits + c] == pb


def test_arrivals_and_manifest_bytes():
    cfg = workloads.c2(seed=3)
    inp = inputs.build_inputs([cfg], mode=_lib.MODE_HISTOGRAM)
    sc = inp.scenarios[0]
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([3, 1])))
    want = list(np.cumsum(rng.exponential(1.0 / cfg.arrival_rate_per_s, size=cfg.clients)))
    assert list(full_pool(inp)[sc.off_arrivals:sc.off_arrivals + cfg.clients]) == want
    prep = oracle.Prepared(cfg)
    assert list(inp.i64[sc.off_manifest:sc.off_manifest + sc.n_seq]) == list(prep.manifest_bytes)


def test_pool_dedup_across_sweep():
    cfgs = [workloads.c3(seed=1, fraction=f / 10) for f in range(11)]
    inp = inputs.build_inputs(cfgs, mode=_lib.MODE_HISTOGRAM)
    offs = {inp.scenarios[i].off_values for i in range(11)}
    assert len(offs) == 1          # one trace table for the whole cache sweep
    caps = [inp.scenarios[i].cache_capacity for i in range(11)]
    assert caps[0] == 1 and caps == sorted(caps)


def test_config_roundtrip_and_fingerprint():
    cfg = ExperimentConfig(variant="TCPF", clients=24, seed=3)
    assert ExperimentConfig.from_dict(cfg.to_dict()) == cfg
    z = workloads.c2()
    d = z.to_dict()
    assert d["experiment"]["popularity"] == "zipf"
    assert ExperimentConfig.from_dict(d).popularity == "zipf"
    # reference-expressible configs carry no extension keys (fingerprint unchanged)
    assert "popularity" not in ExperimentConfig().to_dict()["experiment"]


def test_fingerprint_matches_reference_golden():
    from paper_2603_08417_b200.results import fingerprint
    for name in parity.golden_names():
        _, meta = parity.load_golden(name)
        if meta["popularity"] == "uniform":
            assert fingerprint(ExperimentConfig.from_dict(meta["config"]).to_dict()) == meta["fingerprint"]


def test_validation_errors():
    with pytest.raises(ConfigError):
        ExperimentConfig(variant="TP")
    with pytest.raises(ConfigError):
        ExperimentConfig(clients=0)
    with pytest.raises(ValueError):
        ExperimentConfig(variant="TC", cache_capacity_bytes=0).validate()
    with pytest.raises(ConfigError):
        ExperimentConfig(ladder=[(1, 5), (2, 3)]).validate()


def test_scenario_matrix_grid():
    grid = scenario_matrix(ExperimentConfig())
    assert len(grid) == 72
    assert grid[0][0] == "c04_n1_t2_B"
    assert {c.workers for _, c in grid} == {4, 8}


def test_c5_sweep_shape():
    sweep = workloads.c5_sweep(seeds=range(1, 3))
    assert len(sweep) == 2 * 16
    assert all(len(c.ladder) == 10 for c in sweep)


def _np_gen(ent):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(ent)))


@pytest.mark.parametrize("ent", [[7, 2, 0], [1, 2, 2799], [123456789012, 1], [0], [5, 0], [2**40 + 3, 2, 17]])
def test_host_generator_replays_numpy_streams(ent):
    """otf_np_draws (SeedSequence + PCG64 + numpy's ziggurats, csrc/otf_hostgen.cu) is
    bit-identical to numpy 2.3.5's Generator -- 400k draws per kind, so the
    rejection and tail branches of both ziggurats are exercised."""
    L = _lib.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    e = (ctypes.c_uint64 * len(ent))(*ent)
    n = 400_000
    cases = [(_lib.DRAW_STANDARD_NORMAL, 0.0, 1.0, lambda g: g.standard_normal(n)),
             (_lib.DRAW_NORMAL, 0.0, 0.05, lambda g: g.normal(0.0, 0.05, n)),
             (_lib.DRAW_EXPONENTIAL, 0.0, 0.37, lambda g: g.exponential(0.37, n)),
             (_lib.DRAW_STANDARD_EXPONENTIAL, 0.0, 1.0, lambda g: g.standard_exponential(n))]
    for kind, loc, scale, ref in cases:
        out = np.empty(n)
        _lib.check(L.otf_np_draws(kind, e, len(ent), loc, scale, n, out.ctypes.data_as(dp)), "otf_np_draws")
        want = ref(_np_gen(ent))
        assert np.array_equal(out.view(np.int64), want.view(np.int64)), kind
    z = _np_gen(ent).standard_normal(n)
    assert (np.abs(z) > 3.6541528853610088).sum() > 0      # the tail branch was exercised


def test_host_noise_and_arrivals_tables():
    """otf_gen_noise / otf_gen_arrivals == transcode.py:89-99 / orchestrator.py:265-268 streams."""
    L = _lib.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    eps = np.empty((4, 5000))
    _lib.check(L.otf_gen_noise(11, 4, 0.05, 5000, eps.ctypes.data_as(dp), 3), "otf_gen_noise")
    for w in range(4):
        want = _np_gen([11, w]).normal(0.0, 0.05, size=5000)
        assert np.array_equal(eps[w].view(np.int64), want.view(np.int64))
    arr = np.empty(2800)
    _lib.check(L.otf_gen_arrivals(11, 2800, 1 / 46.0, arr.ctypes.data_as(dp)), "otf_gen_arrivals")
    want = np.cumsum(_np_gen([11, 1]).exponential(1 / 46.0, size=2800))
    assert np.array_equal(arr.view(np.int64), want.view(np.int64))


def test_trace_tables_many_clients_threaded():
    """Multithreaded otf_gen_traces == per-client numpy normals + otf_build_traces."""
    L = _lib.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    n, nc = 600, 300
    starts = np.arange(n, dtype=np.float64)
    mu, sigma, decay = math.log(17e6), 0.35, math.exp(-0.08)
    spread = sigma * math.sqrt(1 - decay * decay)
    v1, p1 = np.empty((nc, n)), np.empty(nc)
    _lib.check(L.otf_gen_traces(9, nc, n, starts.ctypes.data_as(dp), 600.0, mu, sigma, decay, spread, 2e6, 400e6,
                                v1.ctypes.data_as(dp), p1.ctypes.data_as(dp), 8), "otf_gen_traces")
    z = np.stack([_np_gen([9, 2, c]).standard_normal(n + 1) for c in range(nc)])
    v2, p2 = np.empty((nc, n)), np.empty(nc)
    _lib.check(L.otf_build_traces(nc, n, z.ctypes.data_as(dp), starts.ctypes.data_as(dp), 600.0, mu, sigma, decay,
                                  spread, 2e6, 400e6, v2.ctypes.data_as(dp), p2.ctypes.data_as(dp), 1), "b")
    assert np.array_equal(v1.view(np.int64), v2.view(np.int64))
    assert np.array_equal(p1.view(np.int64), p2.view(np.int64))


def test_seed_range_is_validated():
    """Seeds travel as uint64 entropy words (SeedSequence([seed, ...])): out-of-range seeds
    are refused up front instead of being silently truncated."""
    for bad in (-1, 2 ** 64):
        with pytest.raises((ConfigError, ValueError)):
            ExperimentConfig(seed=bad).validate()
    ExperimentConfig(seed=2 ** 64 - 1).validate()


def test_generator_jobs_cover_the_device_prefix():
    """Every device-only f64 element belongs to exactly one generator job, jobs
    start on OTF_GEN_ALIGN boundaries in increasing order, and the host part
    starts after the prefix (only it is copied)."""
    cfgs = workloads.c5_sweep(seeds=range(1, 3))[:8] + [workloads.c2(seed=1), workloads.c1(seed=1)]
    inp = inputs.build_inputs(cfgs, mode=_lib.MODE_HISTOGRAM)
    cover = np.zeros(inp.f64_dev, dtype=np.int32)
    prev_end = 0
    for j in inp.gen_jobs[:inputs.n_gen_jobs(inp)]:
        assert j.first_stream % _lib.GEN_ALIGN == 0 and j.first_stream >= prev_end
        prev_end = j.first_stream + j.n_streams
        n_out = j.n_streams * j.n if j.kind != _lib.GEN_ARRIVALS else j.n
        cover[j.off_out:j.off_out + n_out] += 1
        if j.kind == _lib.GEN_TRACE:
            cover[j.off_pbits:j.off_pbits + j.n_streams] += 1
            assert j.off_starts >= inp.f64_dev                 # starts come from the host part
    assert prev_end == inp.gen_streams
    assert (cover == 1).all()
    for sc in inp.scenarios:
        assert sc.off_values < inp.f64_dev and sc.off_arrivals < inp.f64_dev and sc.off_eps < inp.f64_dev


def test_libm_restatement_matches_host_libm():
    """otf_libm.cuh (host build) == glibc's exp / log1p (math.exp / math.log1p call
    the same libm the reference and numpy use) on the streams' argument ranges,
    random bit patterns and edge cases.  The device build is compared on 1e8
    arguments in tests/test_gpu_gen.py."""
    L = _lib.lib()
    rng = np.random.default_rng(5)
    n = 400_000
    u = rng.random(n)
    xs_exp = np.concatenate([
        13.0 + 8.0 * u,                                   # trace log-bandwidths (mu = log 17e6, sigma 0.35)
        -0.5 * (3.7 * u) ** 2, -7.7 * u,                  # ziggurat wedge tests
        (u - 0.5) * 1500.0, np.ldexp(u - 0.5, -rng.integers(0, 70, n)),
        rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64),
        [0.0, -0.0, 709.78, 709.79, -745.1, -745.2, 1e-300, np.inf, -np.inf]])
    xs_log = np.concatenate([
        -u, -np.ldexp(u, -rng.integers(0, 60, n)), u * 10.0, np.ldexp(u, rng.integers(0, 80, n)),
        -u * 0.999999,
        [0.0, -0.0, -0.29289, -0.2928932188134524, -0.9999999999999999, 0.41421356, 1e-300, np.inf]])
    for fn, xs, ref in ((0, xs_exp, math.exp), (1, xs_log, math.log1p)):
        xs = np.ascontiguousarray(xs[np.isfinite(xs) | np.isinf(xs)])
        out = np.empty_like(xs)
        _lib.check(L.otf_model_libm(fn, xs.ctypes.data, xs.size, out.ctypes.data), "otf_model_libm")
        want = np.empty_like(xs)
        for i, x in enumerate(xs):
            try:
                want[i] = ref(float(x))
            except OverflowError:
                want[i] = np.inf
        bad = np.nonzero(out.view(np.int64) != want.view(np.int64))[0]
        assert bad.size == 0, (fn, xs[bad[:5]], out[bad[:5]], want[bad[:5]])


def test_build_inputs_same_for_configs_and_lowered_memo_cold_and_warm():
    """run_batch lowers each config once and hands the Lowered objects to
    build_inputs, which memoizes the catalog tables per lowering group: the batch
    must be byte-identical to one built from the configs with cold memos."""
    import dataclasses
    cfgs = workloads.c5_sweep(seeds=range(1, 4))
    cfgs += [dataclasses.replace(c, clients=300, zipf_exponent=1.1) for c in cfgs[:5]]

    def blob(inp):
        return (bytes(inp.scenarios), bytes(inp.size_tables), bytes(inp.gen_jobs), inp.f64.tobytes(),
                inp.i64.tobytes(), inp.i32.tobytes(), inp.scratch_bytes, inp.shared_bytes, tuple(inp.smem_per),
                inp.tail_caps.tobytes(), inp.input_bytes)

    for memo in (inputs._LOWER_MEMO, inputs._GRID_MEMO, inputs._SIZE_MEMO, inputs._EPS_MEMO, inputs._MAN_MEMO):
        memo.clear()
    cold = blob(inputs.build_inputs(cfgs, mode=_lib.MODE_HISTOGRAM))
    lows = [inputs.lower_any(c) for c in cfgs]
    assert all(inputs.lower_any(l) is l for l in lows)
    warm = blob(inputs.build_inputs(lows, mode=_lib.MODE_HISTOGRAM))
    assert cold == warm
    again = blob(inputs.build_inputs(list(reversed(lows)), mode=_lib.MODE_HISTOGRAM))
    assert again != warm                               # (order matters: the scenario table is reversed)
    assert blob(inputs.build_inputs(cfgs, mode=_lib.MODE_HISTOGRAM)) == cold
