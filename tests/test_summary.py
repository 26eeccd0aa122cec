"""The histogram-mode summary on CPU: the exact-sum arithmetic of the summary
pass (csrc/otf_xacc.cuh, through the otf_model_exact_sum host hook) against
math.fsum, and the QoE-block -> summary() path against the summaries the
unmodified reference wrote for every golden fixture (orchestrator.py:280-309,
metrics.py:67-116).  The device side of both is in test_gpu_summary.py."""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

from oracle import oracle
from paper_2603_08417_b200 import _lib
from paper_2603_08417_b200.config import ExperimentConfig
from paper_2603_08417_b200.results import ExperimentResult
from tests import parity


def _cfg(meta):
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    cfg.zipf_exponent = meta["zipf_exponent"]
    return cfg


def _xsum(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = ctypes.c_double()
    rc = _lib.lib().otf_model_exact_sum(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(v),
                                        ctypes.byref(out))
    return rc, out.value


@pytest.mark.parametrize("seed", range(6))
def test_exact_sum_is_fsum(seed):
    rng = np.random.default_rng(seed)
    cases = [
        rng.exponential(0.5, 100_000),                              # request-latency-like
        rng.uniform(0, 1, 5000) * 10.0 ** rng.integers(-20, 18, 5000),   # wide exponent spread
        np.concatenate([[2.0 ** 60], np.full(1000, 1.0), [2.0 ** -70]]),   # cancellation-prone order
        np.full(4097, 0.1),
        rng.lognormal(0, 3, 20_000),
    ]
    for v in cases:
        v = v[(v == 0) | ((v >= 2.0 ** -76) & (v < 2.0 ** 64))]
        rc, got = _xsum(v)
        assert rc == 0
        assert got == math.fsum(v.tolist()), (got, math.fsum(v.tolist()))
        rc, got2 = _xsum(v[::-1].copy())                   # order-independent
        assert got2 == got


def test_exact_sum_ties_round_to_even():
    ulp = 2.0 ** -52
    for v in ([1.0, ulp / 2], [1.0 + ulp, ulp / 2], [1.0, ulp / 2, 2.0 ** -70], [3.0, 2.0 ** -51, 2.0 ** -60]):
        assert _xsum(v)[1] == math.fsum(v)


def test_exact_sum_flags_uncovered_values():
    assert _xsum([1.0, 2.0 ** 70])[0] == 1
    assert _xsum([1.0, 1e-300])[0] == 1
    assert _xsum([1.0, 0.0])[0] == 0


@pytest.mark.parametrize("name", parity.golden_names())
def test_qoe_block_summary_is_the_references(name):
    """oracle records -> otf_qoe fields (oracle.qoe_block) -> ExperimentResult.summary()
    in histogram mode == the summary.json the reference wrote, every key exact."""
    _, meta = parity.load_golden(name)
    cfg = _cfg(meta)
    res = oracle.run(cfg)
    q = oracle.qoe_block(res)
    q["summary_flags"] = _lib.Q_ORDER_STATS
    counts = [res["n_req"], res["n_sess"], res["n_seg"], res["n_job"]]
    stats = np.zeros(_lib.ST_NSLOTS, dtype=np.int64)
    stats[:18] = res["stats"][:18]
    r = ExperimentResult(cfg, {}, stats, meta["seq_ids"], qoe=q, counts=counts)
    got, want = r.summary(), dict(meta["summary"])
    if meta["popularity"] != "uniform":                 # Zipf shim: not in the reference's config document
        got.pop("fingerprint"), want.pop("fingerprint")
    assert got == want
