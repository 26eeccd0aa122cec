"""Generate golden fixtures by running the UNMODIFIED reference (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every config in ``tests/golden/cases.py`` this imports
``otfstream.orchestrator.run_experiment`` from /root/reference, runs it, and
stores the result as SoA arrays in ``tests/golden/<name>.npz`` together with
the config document, the backend stats dict and ``ExperimentResult.summary()``.
Zipf-popularity configs (an extension the reference does not have) run the
reference through a shim that replaces only the per-session pick
(orchestrator.py:340-342) by an inverse-CDF draw over ``picks.random()`` from
the same PCG64(SeedSequence([seed, 3, cid])) stream -- see DESIGN.md.
The fixtures are committed; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import json
import logging
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from otfstream import orchestrator as ref_orch  # noqa: E402

import cases  # noqa: E402

PATHS = {"storage": 0, "cache": 1, "waited_inflight": 2, "transcoded": 3, "error": 4}
ORIGINS = {"demand": 0, "speculative": 1}
OUTCOMES = {"pending": 0, "completed": 1, "dropped": 2, "failed": 3}
CSV_CASES = {"grid_c4_k4_t2_T", "edge_two_clients", "edge_short_horizon"}


def zipf_cdf(n, s):
    w = [float(k) ** (-s) for k in range(1, n + 1)]
    acc, c = 0.0, []
    for x in w:
        acc += x
        c.append(acc)
    return [x / acc for x in c]


class _ZipfGenerator:
    """Generator proxy whose integers(n) is a Zipf inverse-CDF pick over random()."""

    def __init__(self, gen, cdf):
        self._g = gen
        self._cdf = cdf

    def integers(self, n):
        u = self._g.random()
        for k, c in enumerate(self._cdf):
            if u < c:
                return k
        return n - 1

    def __getattr__(self, name):
        return getattr(self._g, name)


class _RandomProxy:
    def __init__(self, cdf):
        self._cdf = cdf

    def Generator(self, bitgen):  # noqa: N802 - mirrors numpy's name
        return _ZipfGenerator(np.random.Generator(bitgen), self._cdf)

    def __getattr__(self, name):
        return getattr(np.random, name)


class _NpProxy:
    def __init__(self, cdf):
        self.random = _RandomProxy(cdf)

    def __getattr__(self, name):
        return getattr(np, name)


def run_reference(cfg_doc: dict, popularity: str, zipf_s: float):
    rcfg = ref_orch.ExperimentConfig.from_dict(cfg_doc)
    if popularity == "zipf":
        n = len(rcfg.sequences) if rcfg.sequences else 4
        saved = ref_orch.np
        ref_orch.np = _NpProxy(zipf_cdf(n, zipf_s))
        try:
            return rcfg, ref_orch.run_experiment(rcfg)
        finally:
            ref_orch.np = saved
    return rcfg, ref_orch.run_experiment(rcfg)


def _f(x):
    return float("nan") if x is None else float(x)


def dump(name: str, cfg) -> None:
    doc = cfg.to_dict()
    rcfg, res = run_reference(doc, cfg.popularity, cfg.zipf_exponent)
    seq_ids = [e["id"] for e in rcfg.sequences] if rcfg.sequences else ["longdress", "loot", "redandblack", "soldier"]
    sidx = {s: i for i, s in enumerate(seq_ids)}
    R = res.requests
    arrays = {
        "req_id": np.array([r.request_id for r in R], dtype=np.int64),
        "req_seq": np.array([sidx[r.sequence] for r in R], dtype=np.int32),
        "req_rep": np.array([r.rep for r in R], dtype=np.int32),
        "req_index": np.array([r.index for r in R], dtype=np.int32),
        "req_path": np.array([PATHS[r.path] for r in R], dtype=np.int32),
        "req_arrival": np.array([float(r.arrival_s) for r in R], dtype=np.float64),
        "req_response": np.array([float(r.response_s) for r in R], dtype=np.float64),
        "req_bytes": np.array([r.nbytes for r in R], dtype=np.int64),
    }
    S = res.sessions
    arrays.update({
        "sess_client": np.array([s.client_id for s in S], dtype=np.int32),
        "sess_seq": np.array([sidx[s.sequence] for s in S], dtype=np.int32),
        "sess_stalls": np.array([s.stalls for s in S], dtype=np.int32),
        "sess_flags": np.array([(1 if s.finished else 0) | (2 if s.aborted else 0) for s in S], dtype=np.int32),
        "sess_start": np.array([float(s.start_s) for s in S], dtype=np.float64),
        "sess_end": np.array([float(s.end_s) for s in S], dtype=np.float64),
        "sess_stall_time": np.array([float(s.stall_time_s) for s in S], dtype=np.float64),
        "sess_startup": np.array([_f(s.startup_delay_s) for s in S], dtype=np.float64),
    })
    segs = [(i, g) for i, s in enumerate(S) for g in s.segments]
    arrays.update({
        "seg_session": np.array([i for i, _ in segs], dtype=np.int32),
        "seg_index": np.array([g.index for _, g in segs], dtype=np.int32),
        "seg_rep": np.array([g.rep for _, g in segs], dtype=np.int32),
        "seg_start": np.array([float(g.dl_start_s) for _, g in segs], dtype=np.float64),
        "seg_end": np.array([float(g.dl_end_s) for _, g in segs], dtype=np.float64),
    })
    J = res.jobs
    arrays.update({
        "job_seq": np.array([sidx[j.target.sequence] for j in J], dtype=np.int32),
        "job_rep": np.array([j.target.rep for j in J], dtype=np.int32),
        "job_index": np.array([j.target.index for j in J], dtype=np.int32),
        "job_origin": np.array([ORIGINS[j.origin] for j in J], dtype=np.int32),
        "job_outcome": np.array([OUTCOMES[j.outcome] for j in J], dtype=np.int32),
        "job_enq": np.array([_f(j.enqueued_at) for j in J], dtype=np.float64),
        "job_start": np.array([_f(j.started_at) for j in J], dtype=np.float64),
        "job_fin": np.array([_f(j.finished_at) for j in J], dtype=np.float64),
    })
    summary = res.summary()
    meta = {
        "name": name,
        "config": doc,
        "popularity": cfg.popularity,
        "zipf_exponent": cfg.zipf_exponent,
        "fingerprint": res.fingerprint,
        "backend_stats": res.backend_stats,
        "summary": json.loads(json.dumps(summary, default=float)),
        "seq_ids": seq_ids,
    }
    arrays["meta"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode("utf-8"), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    if name in CSV_CASES:                               # the reference's own on-disk bundle
        res.write(os.path.join(HERE, "csv", name))
    print(f"{name}: requests {len(R)} sessions {len(S)} jobs {len(J)}")


def matrix_bundles():
    """Reference CSV bundles of two grid points of scenario_matrix(ExperimentConfig())."""
    grid = dict(ref_orch.scenario_matrix(ref_orch.ExperimentConfig()))
    for name in ("c24_n1_t4_TCPF", "c04_n2_t2_TC"):
        ref_orch.run_experiment(grid[name]).write(os.path.join(HERE, "csv_matrix", name))
        print("matrix bundle", name)


def main(argv):
    logging.disable(logging.WARNING)
    if argv[1:] == ["matrix"]:
        matrix_bundles()
        return
    only = set(argv[1:])
    for name, cfg in cases.golden_cases():
        if only and name not in only:
            continue
        dump(name, cfg)


if __name__ == "__main__":
    main(sys.argv)
