"""TEST INFRASTRUCTURE ONLY -- Python driver for the C oracle (otf_oracle.c).

The oracle is a CPU restatement of the reference's ``run_experiment``
(/root/reference/pkg/src/otfstream/orchestrator.py:327-370).  This module
derives the reference's seeded random streams with numpy exactly where the
reference draws them and hands everything else to C:

* arrival draws   -- orchestrator.py:265-268  (exponential, SS([seed, 1]))
* trace normals   -- orchestrator.py:254-263 + netem.py:179-202 (SS([seed, 2, cid]))
* worker noise    -- transcode.py:89-99 (SS([seed, worker_id]))
* sequence keys   -- content.py:165-167 (sha256(id)[:8], big-endian)
* manifest bytes  -- server.py:58-59 (len(json.dumps(manifest, sort_keys=True)))

Segment sizes (SeedSequence + PCG64 + uniform) and sequence picks (PCG64
integers / random) are restated in C.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

PATHS = ("storage", "cache", "waited_inflight", "transcoded", "error")
ORIGINS = ("demand", "speculative")
OUTCOMES = ("pending", "completed", "dropped", "failed")
SKIP_REASONS = ("disabled", "end-of-sequence", "stored", "cached", "in-flight", "overload")
FIXTURE_SEQUENCES = ["longdress", "loot", "redandblack", "soldier"]

ST = dict(jobs_total=0, jobs_demand=1, jobs_speculative=2, wasted_avoided=3, speculation_enqueued=4,
          skip0=5, capacity_bytes=11, current_bytes=12, entries=13, hits=14, misses=15,
          evictions=16, rejected=17, status=18, hung=19, timer_pops=20, ready_callbacks=21)

_P = ctypes.POINTER


class Scenario(ctypes.Structure):
    _fields_ = [
        ("n_clients", ctypes.c_int32), ("n_workers", ctypes.c_int32), ("n_seq", ctypes.c_int32),
        ("n_ranks", ctypes.c_int32), ("max_nseg", ctypes.c_int32), ("n_samples", ctypes.c_int32),
        ("cache_enabled", ctypes.c_int32), ("spec_enabled", ctypes.c_int32),
        ("popularity", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("stored_mask", ctypes.c_uint32), ("pad1", ctypes.c_uint32),
        ("cache_capacity", ctypes.c_int64),
        ("seed", ctypes.c_uint64), ("catalog_seed", ctypes.c_uint64),
        ("horizon", ctypes.c_double), ("latency", ctypes.c_double), ("target", ctypes.c_double),
        ("safe", ctypes.c_double), ("panic", ctypes.c_double), ("resume", ctypes.c_double),
        ("startup", ctypes.c_double), ("alpha", ctypes.c_double), ("headroom", ctypes.c_double),
        ("noise", ctypes.c_double), ("size_jitter", ctypes.c_double),
        ("trace_mu", ctypes.c_double), ("trace_sigma", ctypes.c_double),
        ("trace_decay", ctypes.c_double), ("trace_spread", ctypes.c_double),
        ("trace_floor", ctypes.c_double), ("trace_cap", ctypes.c_double),
        ("trace_step", ctypes.c_double), ("trace_duration", ctypes.c_double),
        ("bitrates", _P(ctypes.c_int64)), ("rho", _P(ctypes.c_double)),
        ("seq_duration", _P(ctypes.c_double)), ("seq_segdur", _P(ctypes.c_double)),
        ("seq_key", _P(ctypes.c_int64)), ("manifest_bytes", _P(ctypes.c_int64)),
        ("arrival_draws", _P(ctypes.c_double)), ("trace_normals", _P(ctypes.c_double)),
        ("zipf_cdf", _P(ctypes.c_double)), ("eps", _P(ctypes.c_double)),
        ("eps_per_worker", ctypes.c_int64),
        ("queue_bound", ctypes.c_int32), ("retries", ctypes.c_int32), ("retry_backoff", ctypes.c_double),
        ("demand_priority", ctypes.c_int32), ("pad2", ctypes.c_int32),
        ("tr_starts", _P(ctypes.c_double)), ("tr_values", _P(ctypes.c_double)),
        ("tr_period", _P(ctypes.c_double)), ("tr_pbits", _P(ctypes.c_double)),
        ("tr_off", _P(ctypes.c_int64)), ("tr_n", _P(ctypes.c_int32)),
    ]


_OUT_ARRAYS = [
    ("req_id", np.int64), ("req_seq", np.int32), ("req_rep", np.int32), ("req_index", np.int32),
    ("req_path", np.int32), ("req_arrival", np.float64), ("req_response", np.float64),
    ("req_bytes", np.int64),
    ("sess_client", np.int32), ("sess_seq", np.int32), ("sess_stalls", np.int32),
    ("sess_flags", np.int32), ("sess_start", np.float64), ("sess_end", np.float64),
    ("sess_stall_time", np.float64), ("sess_startup", np.float64),
    ("seg_session", np.int32), ("seg_index", np.int32), ("seg_rep", np.int32),
    ("seg_start", np.float64), ("seg_end", np.float64),
    ("job_seq", np.int32), ("job_rep", np.int32), ("job_index", np.int32), ("job_origin", np.int32),
    ("job_outcome", np.int32), ("job_enq", np.float64), ("job_start", np.float64),
    ("job_fin", np.float64),
]
_CT = {np.int64: ctypes.c_int64, np.int32: ctypes.c_int32, np.float64: ctypes.c_double}


class Outputs(ctypes.Structure):
    _fields_ = ([("req_cap", ctypes.c_int64), ("sess_cap", ctypes.c_int64),
                 ("seg_cap", ctypes.c_int64), ("job_cap", ctypes.c_int64)]
                + [(n, _P(_CT[t])) for n, t in _OUT_ARRAYS]
                + [("n_req", ctypes.c_int64), ("n_sess", ctypes.c_int64),
                   ("n_seg", ctypes.c_int64), ("n_job", ctypes.c_int64),
                   ("stats", ctypes.c_int64 * 32)])


_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so in place (oracle/Makefile)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "otf_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.oracle_run.argtypes = [_P(Scenario), _P(Outputs)]
        _lib.oracle_libm.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_segment_sizes.argtypes = [_P(Scenario), _P(ctypes.c_int64), _P(ctypes.c_int32)]
        _lib.oracle_build_traces.argtypes = [_P(Scenario), _P(ctypes.c_double),
                                             _P(ctypes.c_double), _P(ctypes.c_double)]
        _lib.oracle_sample_times.argtypes = [ctypes.c_double, ctypes.c_double,
                                             _P(ctypes.c_double), ctypes.c_int]
        _lib.oracle_sample_times.restype = ctypes.c_int
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(_P(ct))


def _gen(entropy):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


def zipf_cdf(n: int, s: float) -> np.ndarray:
    """Normalised cumulative Zipf(s) weights over ranks 1..n (extension)."""
    w = [float(k) ** (-s) for k in range(1, n + 1)]
    acc, c = 0.0, []
    for x in w:
        acc += x
        c.append(acc)
    return np.array([x / acc for x in c], dtype=np.float64)


def load_trace_csv(path):
    """netem.load_trace + BandwidthTrace.__init__ (netem.py:148-161, 39-64), restated."""
    import csv
    import statistics
    samples = []
    with open(path, newline="", encoding="utf-8") as fh:
        for row in csv.reader(fh):
            if not row or row[0].lstrip().startswith("#"):
                continue
            try:
                ts, kbps = float(row[0]), float(row[1])
            except ValueError:
                continue
            samples.append((ts, kbps * 1000.0))
    if not samples:
        raise ValueError(f"no samples in trace file {path}")
    ts = [t for t, _ in samples]
    if any(b - a <= 0 for a, b in zip(ts, ts[1:])) or ts[0] < 0 or any(bw < 0 for _, bw in samples):
        raise ValueError(f"invalid trace {path}")
    starts = list(ts)
    values = [float(bw) for _, bw in samples]
    if starts[0] > 0:
        starts[0] = 0.0
    gaps = [b - a for a, b in zip(ts, ts[1:])]
    period = ts[-1] + (statistics.median(gaps) if gaps else 1.0)
    pbits = sum(v * ((starts[i + 1] if i + 1 < len(starts) else period) - starts[i]) for i, v in enumerate(values))
    return starts, values, period, pbits


def _attr(cfg, name, default):
    return getattr(cfg, name, default)


class Prepared:
    """Every input array the C oracle needs for one config (kept alive for ctypes)."""

    def __init__(self, cfg, eps_per_worker: int | None = None):
        self.cfg = cfg
        ladder = sorted(cfg.ladder)
        n_ranks = len(ladder)
        variant = cfg.variant.replace("+", "").upper()
        if variant == "B":
            stored = list(range(1, n_ranks + 1))
        elif "F" in variant:
            stored = [1, n_ranks]
        else:
            stored = [n_ranks]
        entries = cfg.sequences or [{"id": sid} for sid in FIXTURE_SEQUENCES]
        seqs = [(e["id"], float(e.get("duration_s", cfg.sequence_duration_s)),
                 float(e.get("segment_duration_s", cfg.segment_duration_s))) for e in entries]
        self.seq_ids = [s[0] for s in seqs]
        counts = [math.ceil(d / t) for _, d, t in seqs]
        self.counts = counts
        n_seq = len(seqs)
        ne = cfg.netem
        self.bitrates = np.array([b for _, b in ladder], dtype=np.int64)
        rho_map = cfg.per_rank_rho or {r: cfg.rho for r, _ in ladder}
        self.rho = np.array([float(rho_map[r]) for r, _ in ladder], dtype=np.float64)
        self.seq_duration = np.array([s[1] for s in seqs], dtype=np.float64)
        self.seq_segdur = np.array([s[2] for s in seqs], dtype=np.float64)
        self.seq_key = np.array([int.from_bytes(hashlib.sha256(s[0].encode("utf-8")).digest()[:8], "big")
                                 for s in seqs], dtype=np.uint64).view(np.int64)
        man = []
        for (sid, dur, segdur), cnt in zip(seqs, counts):
            m = {"sequence": sid, "duration_s": dur, "segment_duration_s": segdur,
                 "segment_count": cnt,
                 "representations": [{"rank": r, "bitrate_bps": b} for r, b in ladder],
                 "url_template": "/content/{seq}/{rep}/{index}"}
            man.append(len(json.dumps(m, sort_keys=True).encode("utf-8")))
        self.manifest_bytes = np.array(man, dtype=np.int64)
        N, K = cfg.clients, cfg.workers
        self.arrival_draws = _gen([cfg.seed, 1]).exponential(1.0 / cfg.arrival_rate_per_s, size=N)
        nsamp = 0
        t = 0.0
        while t < ne.trace_duration_s:
            nsamp += 1
            t += ne.step_s
        self.n_samples = nsamp
        self.trace_normals = np.empty((N, nsamp + 1), dtype=np.float64)
        self.csv = None
        if ne.trace_dir:                               # orchestrator.py:243-253
            files = sorted(os.path.join(ne.trace_dir, f) for f in os.listdir(ne.trace_dir) if f.endswith(".csv"))
            order = _gen([cfg.seed, 2]).permutation(len(files))
            tabs = [load_trace_csv(f) for f in files]
            st, vv, off, nn, per, pb = [], [], [], [], [], []
            pos = 0
            for c in range(N):
                s_, v_, p_, b_ = tabs[order[c % len(files)]]
                off.append(pos); nn.append(len(s_)); per.append(p_); pb.append(b_)
                st.extend(s_); vv.extend(v_); pos += len(s_)
            self.csv = (np.array(st), np.array(vv), np.array(per), np.array(pb),
                        np.array(off, dtype=np.int64), np.array(nn, dtype=np.int32))
        else:
            for c in range(N):
                self.trace_normals[c] = _gen([cfg.seed, 2, c]).standard_normal(nsamp + 1)
        pop = _attr(cfg, "popularity", "uniform")
        self.zipf = zipf_cdf(n_seq, float(_attr(cfg, "zipf_exponent", 0.8))) \
            if pop == "zipf" else np.zeros(n_seq)
        if eps_per_worker is None:
            eps_per_worker = 64 + int(4 * N * cfg.horizon_s / max(min(s[2] for s in seqs), 1e-3) / K)
        self.eps_per_worker = eps_per_worker
        if cfg.noise_rel_std > 0:
            self.eps = np.stack([_gen([cfg.seed, w]).normal(0.0, cfg.noise_rel_std, size=eps_per_worker)
                                 for w in range(K)])
        else:
            self.eps = np.zeros((K, 1))
        self.max_nseg = max(counts)
        median = ne.median_bps
        decay = math.exp(-ne.theta_per_s * ne.step_s)
        sc = Scenario()
        sc.n_clients, sc.n_workers, sc.n_seq, sc.n_ranks = N, K, n_seq, n_ranks
        sc.max_nseg, sc.n_samples = self.max_nseg, nsamp
        sc.cache_enabled = int("C" in variant)
        sc.spec_enabled = int("P" in variant)
        sc.popularity = 1 if pop == "zipf" else 0
        sc.stored_mask = sum(1 << r for r in stored)
        sc.cache_capacity = int(cfg.cache_capacity_bytes)
        sc.seed = cfg.seed
        sc.catalog_seed = cfg.seed
        sc.horizon = float(cfg.horizon_s)
        sc.latency = float(cfg.client.latency_s)
        b = cfg.client.buffer
        sc.target, sc.safe, sc.panic, sc.resume, sc.startup = b.target_s, b.safe_s, b.panic_s, b.resume_s, b.startup_s
        sc.alpha, sc.headroom = cfg.client.ewma_alpha, cfg.client.headroom
        sc.noise = cfg.noise_rel_std
        sc.size_jitter = cfg.size_jitter
        sc.trace_mu = math.log(median)
        sc.trace_sigma = ne.sigma
        sc.trace_decay = decay
        sc.trace_spread = ne.sigma * math.sqrt(1.0 - decay * decay)
        sc.trace_floor, sc.trace_cap = ne.floor_bps, ne.cap_bps
        sc.trace_step, sc.trace_duration = ne.step_s, ne.trace_duration_s
        sc.bitrates = _ptr(self.bitrates, ctypes.c_int64)
        sc.rho = _ptr(self.rho, ctypes.c_double)
        sc.seq_duration = _ptr(self.seq_duration, ctypes.c_double)
        sc.seq_segdur = _ptr(self.seq_segdur, ctypes.c_double)
        sc.seq_key = _ptr(self.seq_key, ctypes.c_int64)
        sc.manifest_bytes = _ptr(self.manifest_bytes, ctypes.c_int64)
        sc.arrival_draws = _ptr(self.arrival_draws, ctypes.c_double)
        sc.trace_normals = _ptr(self.trace_normals, ctypes.c_double)
        sc.zipf_cdf = _ptr(self.zipf, ctypes.c_double)
        sc.eps = _ptr(self.eps, ctypes.c_double)
        sc.eps_per_worker = self.eps.shape[1]
        sc.queue_bound = int(cfg.queue_bound)
        sc.retries = int(cfg.client.retries)
        sc.retry_backoff = float(cfg.client.retry_backoff_s)
        sc.demand_priority = int(bool(cfg.demand_priority))
        if self.csv is not None:
            st, vv, per, pb, off, nn = self.csv
            sc.tr_starts, sc.tr_values = _ptr(st, ctypes.c_double), _ptr(vv, ctypes.c_double)
            sc.tr_period, sc.tr_pbits = _ptr(per, ctypes.c_double), _ptr(pb, ctypes.c_double)
            sc.tr_off, sc.tr_n = _ptr(off, ctypes.c_int64), _ptr(nn, ctypes.c_int32)
        self.sc = sc

    def sizes(self):
        n = self.sc.n_seq * self.sc.n_ranks * self.sc.max_nseg
        sizes = np.zeros(n, dtype=np.int64)
        counts = np.zeros(self.sc.n_seq, dtype=np.int32)
        lib().oracle_segment_sizes(ctypes.byref(self.sc), _ptr(sizes, ctypes.c_int64),
                                   _ptr(counts, ctypes.c_int32))
        return sizes.reshape(self.sc.n_seq, self.sc.n_ranks, self.sc.max_nseg), counts

    def traces(self):
        N, n = self.sc.n_clients, self.sc.n_samples
        values = np.zeros((N, n), dtype=np.float64)
        pbits = np.zeros(N, dtype=np.float64)
        period = np.zeros(1, dtype=np.float64)
        lib().oracle_build_traces(ctypes.byref(self.sc), _ptr(values, ctypes.c_double),
                                  _ptr(pbits, ctypes.c_double), _ptr(period, ctypes.c_double))
        starts = np.zeros(n, dtype=np.float64)
        lib().oracle_sample_times(self.sc.trace_duration, self.sc.trace_step,
                                  _ptr(starts, ctypes.c_double), n)
        return starts, values, pbits, float(period[0])


def run(cfg, caps=None, eps_per_worker=None) -> dict:
    """Run the oracle for one config; returns SoA numpy arrays + stats."""
    prep = Prepared(cfg, eps_per_worker)
    if caps is None:
        est = int(cfg.clients * cfg.horizon_s * 2 / max(prep.seq_segdur.min(), 1e-3)) + 1024
        caps = dict(req=est, sess=est, seg=est, job=est)
    while True:
        arrays = {}
        out = Outputs()
        out.req_cap, out.sess_cap, out.seg_cap, out.job_cap = caps["req"], caps["sess"], caps["seg"], caps["job"]
        for name, t in _OUT_ARRAYS:
            a = np.zeros(caps[name.split("_")[0]], dtype=t)
            arrays[name] = a
            setattr(out, name, _ptr(a, _CT[t]))
        rc = lib().oracle_run(ctypes.byref(prep.sc), ctypes.byref(out))
        if rc == 0:
            break
        caps = {k: v * 2 for k, v in caps.items()}
    res = {"n_req": out.n_req, "n_sess": out.n_sess, "n_seg": out.n_seg, "n_job": out.n_job}
    for name, _ in _OUT_ARRAYS:
        key = name.split("_")[0]
        n = {"req": out.n_req, "sess": out.n_sess, "seg": out.n_seg, "job": out.n_job}[key]
        res[name] = arrays[name][:n].copy()
    res["stats"] = np.array(list(out.stats), dtype=np.int64)
    res["seq_ids"] = prep.seq_ids
    return res


def backend_stats(res: dict, cache_enabled: bool) -> dict:
    """The reference's Backend.stats() dict (backend.py:228-239) from oracle stats."""
    st = res["stats"]
    skipped = {r: int(st[ST["skip0"] + i]) for i, r in enumerate(SKIP_REASONS) if st[ST["skip0"] + i]}
    out = {
        "jobs_total": int(st[0]), "jobs_demand": int(st[1]), "jobs_speculative": int(st[2]),
        "wasted_avoided": int(st[3]), "speculation_enqueued": int(st[4]),
        "speculation_skipped": skipped,
    }
    if cache_enabled:
        out["cache"] = {k: int(st[ST[k]]) for k in
                        ("capacity_bytes", "current_bytes", "entries", "hits", "misses", "evictions", "rejected")}
    return out


# ---- the fused QoE block (include/otfgpu.h otf_qoe) restated from records -------------
LAT_BINS, STALL_BINS, RANK_BINS = 64, 32, 32
_LAT_EDGES = np.array([(0.01 * (1.0 + 0.25 * (k & 3))) * 2.0 ** (k >> 2) for k in range(LAT_BINS - 1)])


def lat_bins(lat: np.ndarray) -> np.ndarray:
    """Latency histogram bin: 0 = instant (< 10 ms, metrics.py:38,77), then 4 bins per
    octave with lower edges 0.01 * (1 + q/4) * 2^o (csrc/otf_model.cuh lat_bin)."""
    k = np.searchsorted(_LAT_EDGES, lat, side="right") - 1
    return np.where(lat < 0.010, 0, 1 + np.clip(k, 0, LAT_BINS - 2))


def qoe_block(res: dict) -> dict:
    """Every otf_qoe field from one run's records (registration / response order):
    the counters and histograms, the reference's summary statistics
    (orchestrator.py:280-309, metrics.py:67-116: sorted latencies at n // 2 and
    min(n - 1, int(0.99 n)), the left-to-right stall-time sum in registration
    order) and the exact sums (math.fsum) of latencies and startup delays."""
    lat = res["req_response"] - res["req_arrival"]
    n = len(lat)
    stalls = np.asarray(res["sess_stalls"], dtype=np.int64)
    st = np.asarray(res["sess_stall_time"], dtype=np.float64)
    su = np.asarray(res["sess_startup"], dtype=np.float64)
    total = 0.0
    for x in st[st != 0.0]:                            # registration order, plain double adds
        total += float(x)
    srt = np.sort(lat)
    return {
        "lat_hist": [int(x) for x in np.bincount(lat_bins(lat), minlength=LAT_BINS)],
        "path_count": [int((res["req_path"] == p).sum()) for p in range(5)],
        "stall_hist": [int(x) for x in np.bincount(np.minimum(stalls, STALL_BINS - 1), minlength=STALL_BINS)],
        "rank_count": [int(x) for x in np.bincount(np.minimum(res["seg_rep"], RANK_BINS - 1), minlength=RANK_BINS)],
        "n_requests": n, "n_sessions": len(stalls), "n_segments": len(res["seg_rep"]),
        "n_finished": int((np.asarray(res["sess_flags"]) & 1).sum()), "n_started": int((~np.isnan(su)).sum()),
        "n_stalls": int(stalls.sum()),
        "latency_sum": math.fsum(lat.tolist()),
        "stall_time_sum": total,
        "startup_delay_sum": math.fsum(su[~np.isnan(su)].tolist()),
        "latency_p50": float(srt[n // 2]) if n else 0.0,
        "latency_p99": float(srt[min(n - 1, int(0.99 * n))]) if n else 0.0,
        "n_lat_tail": int((lat != 0.0).sum()), "n_stall_tail": int((st != 0.0).sum()),
    }


def run_qoe(cfg) -> dict:
    """oracle run -> its QoE block plus the backend stats row (pool-friendly: small result)."""
    r = run(cfg)
    q = qoe_block(r)
    q["stats"] = [int(x) for x in r["stats"][:18]]
    q["n_job"] = int(r["n_job"])
    return q
