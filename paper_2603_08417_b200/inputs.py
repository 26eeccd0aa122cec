"""Host input builder: lowers ExperimentConfigs to otf_scenario structs + shared pools.

Everything a scenario reads is derived from the reference's own seeded
streams.  The numpy Generator streams are replayed bit-for-bit ON THE DEVICE
(csrc/otf_gen.cu: SeedSequence + PCG64 + numpy's ziggurats + glibc's exp and
log1p), where the reference draws them:

* arrival offsets  list(np.cumsum(exponential(1/rate, N)))  SS([seed, 1])   orchestrator.py:265-268
* trace normals    standard_normal per client               SS([seed, 2, c]) orchestrator.py:254-263
                   -> values/period-bits (glibc exp, CPython 3.12 sum)  netem.py:39-64,179-202
* worker noise     normal(0, noise) per worker              SS([seed, w])    transcode.py:89-99
* segment sizes    uniform jitter per (seq, rank, index)                     content.py:204-218
* session picks    integers(n) / Zipf inverse CDF per client (engine)        orchestrator.py:340-342

The host only lowers the configs and computes what needs no stream:

* sequence keys    sha256(id)[:8] big-endian                                  content.py:165-166
* manifest bytes   len(json.dumps(manifest_for(seq), sort_keys=True))         server.py:58-59

The f64 pool's leading `f64_dev` elements are device-only: the generator jobs
(`gen_jobs`, otf_gen_tables) fill them on the GPU, and only the rest of the
pool is copied from the host.  Tables are de-duplicated across the batch:
traces by (seed, netem), sizes by catalog, arrivals by (seed, N, rate), noise
by (seed, noise), so a sweep over variants / cache sizes / client counts pays
for each stream once.  `host_generate` replays the same jobs with the host
generators (csrc/otf_hostgen.cu) for the tests.
"""

from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import json
import math
import os
import statistics

import numpy as np

from . import _lib
from .config import ExperimentConfig, ConfigError

__all__ = ["BatchInputs", "build_inputs", "zipf_cdf", "sample_times"]

URL_TEMPLATE = "/content/{seq}/{rep}/{index}"


def _gen(entropy):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


def zipf_cdf(n: int, s: float) -> np.ndarray:
    """Normalised cumulative Zipf(s) weights over catalog ranks 1..n (extension)."""
    w = [float(k) ** (-s) for k in range(1, n + 1)]
    acc, c = 0.0, []
    for x in w:
        acc += x
        c.append(acc)
    return np.array([x / acc for x in c], dtype=np.float64)


def load_trace_csv(path: str):
    """netem.load_trace + BandwidthTrace.__init__ (netem.py:148-161, 39-64): the
    (starts, values, period, period_bits) of one CSV trace (timestamp_s, kbps)."""
    import csv
    samples = []
    with open(path, newline="", encoding="utf-8") as fh:
        for row in csv.reader(fh):
            if not row or row[0].lstrip().startswith("#"):
                continue
            try:
                ts, kbps = float(row[0]), float(row[1])
            except ValueError:
                continue                               # header row
            samples.append((ts, kbps * 1000.0))
    if not samples:
        raise ValueError(f"no samples in trace file {path}")
    ts = [t for t, _ in samples]
    if any(b - a <= 0 for a, b in zip(ts, ts[1:])):
        raise ValueError("trace timestamps must strictly increase")
    if ts[0] < 0:
        raise ValueError("trace timestamps must be >= 0")
    if any(bw < 0 for _, bw in samples):
        raise ValueError("bandwidth must be >= 0")
    starts = list(ts)
    values = [float(bw) for _, bw in samples]
    if starts[0] > 0:
        starts[0] = 0.0
    gaps = [b - a for a, b in zip(ts, ts[1:])]
    period = ts[-1] + (statistics.median(gaps) if gaps else 1.0)
    pbits = sum(v * ((starts[i + 1] if i + 1 < len(starts) else period) - starts[i])   # CPython 3.12 sum
                for i, v in enumerate(values))
    return starts, values, period, pbits


def sample_times(duration: float, step: float) -> list[float]:
    """synthetic_trace's timestamps: t = 0; while t < duration: t += step (netem.py:195-201)."""
    ts, t = [], 0.0
    while t < duration:
        ts.append(t)
        t += step
    return ts


@dataclasses.dataclass
class Lowered:
    cfg: ExperimentConfig
    seq_ids: list[str]
    seq_dur: list[float]
    seq_segdur: list[float]
    counts: list[int]
    n_ranks: int
    stored: list[int]
    cache_enabled: bool
    spec_enabled: bool
    cat_key: tuple = ()         # (seed, jitter, ids, durations, segment durations, ladder): one size table

_LOWER_MEMO: dict = {}


def _netem_key(ne) -> tuple:
    return tuple(ne.__dict__.values())                 # NetemConfig: flat scalar fields


def _lower_key(cfg: ExperimentConfig):
    """Every field validate() and the catalog read: configs of a sweep that differ
    only in client count, horizon, cache size within the policy's limits... share
    one validated lowering."""
    seqs = tuple([(e["id"], e.get("duration_s"), e.get("segment_duration_s")) for e in cfg.sequences]) \
        if cfg.sequences else None
    return (cfg.variant, cfg.cache_capacity_bytes > 0, cfg.workers, cfg.queue_bound, cfg.demand_priority,
            tuple(tuple(x) for x in cfg.ladder), seqs, cfg.seed, cfg.size_jitter, cfg.rho,
            tuple(sorted((cfg.per_rank_rho or {}).items())), cfg.noise_rel_std, cfg.clock, cfg.client.retries,
            cfg.segment_duration_s, cfg.sequence_duration_s)


def lower(cfg: ExperimentConfig) -> Lowered:
    """Validate (the reference's constructor checks) and lower one config; the
    catalog part is shared by every config with the same _lower_key."""
    key = _lower_key(cfg)
    hit = _LOWER_MEMO.get(key)
    if hit is not None:
        if not 0 <= int(cfg.seed) < 2 ** 64:           # (part of the key; kept for clarity)
            raise ConfigError("seed must be in [0, 2**64) for the GPU engine")
        return dataclasses.replace(hit, cfg=cfg)
    cfg.validate()
    cat = cfg.catalog_config()
    policy = cfg.policy()
    seqs = cat.sequences
    low = Lowered(
        cfg=cfg,
        seq_ids=[s.id for s in seqs],
        seq_dur=[s.duration_s for s in seqs],
        seq_segdur=[s.segment_duration_s for s in seqs],
        counts=[math.ceil(s.duration_s / s.segment_duration_s) for s in seqs],
        n_ranks=len(cfg.ladder),
        stored=list(cat.stored_ranks),
        cache_enabled=policy.cache_enabled,
        spec_enabled=policy.speculative_enabled,
    )
    low.cat_key = (cfg.seed, cfg.size_jitter, tuple(low.seq_ids), tuple(low.seq_dur), tuple(low.seq_segdur),
                   tuple(sorted(tuple(x) for x in cfg.ladder)))
    if len(_LOWER_MEMO) > 65536:
        _LOWER_MEMO.clear()
    _LOWER_MEMO[key] = low
    return low


def lower_any(c) -> Lowered:
    """lower() of a config of either package, or a config already lowered (run_batch
    lowers each config once per call)."""
    return c if isinstance(c, Lowered) else lower(ExperimentConfig.from_reference(c))


_GRID_MEMO: dict = {}


def _trace_grid(duration: float, step: float):
    """A synthetic trace's sample times, period and grid step (0 if the times are not
    i * step exactly), shared by every (seed, client) with the same netem timing."""
    key = (duration, step)
    hit = _GRID_MEMO.get(key)
    if hit is None:
        ts = sample_times(duration, step)
        if not ts:
            raise ConfigError("trace has no samples")
        gaps = [b - a for a, b in zip(ts, ts[1:])]
        period = ts[-1] + (statistics.median(gaps) if gaps else 1.0)
        grid = float(step) if all(x == float(i) * step for i, x in enumerate(ts)) else 0.0
        if len(_GRID_MEMO) > 256:
            _GRID_MEMO.clear()
        hit = _GRID_MEMO[key] = (ts, period, grid)
    return hit


_SIZE_MEMO: dict = {}


def _engine_bytes(engine: int, N: int, K: int, n_seq: int, n_ranks: int, max_nseg: int, lc: int):
    """(global scratch, shared memory per CTA) of one scenario (memoized C-ABI queries)."""
    key = (engine, N, K, n_seq, n_ranks, max_nseg, lc)
    hit = _SIZE_MEMO.get(key)
    if hit is None:
        L = _lib.lib()
        scratch = int(L.otf_scratch_bytes(engine, N, K, n_seq, n_ranks, max_nseg))
        smem = int(L.otf_shared_bytes_cap(N, n_seq, n_ranks, max_nseg, lc)) if engine == _lib.ENGINE_WINDOWED else 0
        if len(_SIZE_MEMO) > 65536:
            _SIZE_MEMO.clear()
        hit = _SIZE_MEMO[key] = (scratch, smem)
    return hit


class _Pools:
    def __init__(self, threads: int = 1):
        self.threads = threads
        self.parts = {"f64": [], "i64": [], "i32": []}
        self.size = {"f64": 0, "i64": 0, "i32": 0}
        self.dev = {"f64": 0, "i64": 0, "i32": 0}      # device-only prefix (generated on the GPU)
        self.memo = {}

    def device(self, kind: str, n: int) -> int:
        """Reserve n device-only elements (filled by a generator job, never copied)."""
        if self.parts[kind]:
            raise AssertionError("device-only regions must precede every host part")
        off = self.dev[kind]
        self.dev[kind] += int(n)
        self.size[kind] += int(n)
        return off

    def add(self, kind: str, arr, key=None) -> int:
        if key is not None and (kind, key) in self.memo:
            return self.memo[(kind, key)]
        dt = {"f64": np.float64, "i64": np.int64, "i32": np.int32}[kind]
        a = np.ascontiguousarray(np.asarray(arr, dtype=dt).reshape(-1))
        off = self.size[kind]
        self.parts[kind].append(a)
        self.size[kind] += a.size
        if key is not None:
            self.memo[(kind, key)] = off
        return off

    def reserve(self, kind: str, n: int, key=None) -> int:
        return self.add(kind, np.zeros(n), key)

    def concat(self, kind: str, pin: bool = False) -> np.ndarray:
        """The pool as one array (page-locked when pin, so the H2D copy is a single DMA)."""
        dt = {"f64": np.float64, "i64": np.int64, "i32": np.int32}[kind]
        total = max(1, self.size[kind] - self.dev[kind])      # the host part only
        if pin:
            import torch
            tt = {"f64": torch.float64, "i64": torch.int64, "i32": torch.int32}[kind]
            out = torch.empty(total, dtype=tt, pin_memory=True).numpy()
        else:
            out = np.empty(total, dtype=dt)
        pos = 0
        for part in self.parts[kind]:
            out[pos:pos + part.size] = part
            pos += part.size
        out[pos:] = 0
        return out


@dataclasses.dataclass
class BatchInputs:
    lowered: list[Lowered]
    scenarios: ctypes.Array
    size_tables: ctypes.Array
    f64: np.ndarray
    i64: np.ndarray
    i32: np.ndarray
    scratch_bytes: int
    caps: np.ndarray            # [n][4] record capacities (req, sess, seg, job)
    rec_offsets: np.ndarray     # [n][4]
    rec_totals: list[int]       # pool lengths (req, sess, seg, job)
    engine: int
    mode: int
    input_bytes: int            # algorithmic input bytes (for the roofline)
    shared_bytes: int = 0       # windowed engine: dynamic shared memory per CTA (batch max)
    smem_per: list = dataclasses.field(default_factory=list)   # per scenario
    engine_flags: int = 0       # OTF_BF_*
    pinned: bool = False        # pools allocated page-locked (torch pinned memory)
    tail_caps: np.ndarray = None      # [n][4] summary tails: nonzero latencies, sessions, stalled, startups
    tail_totals: tuple = (0, 0, 0)    # pool lengths: latency doubles, session entries, startup doubles
    f64_dev: int = 0                  # leading f64 pool elements generated on the device (not in `f64`)
    gen_jobs: ctypes.Array = None     # otf_gen_job[] (device request generation)
    gen_streams: int = 0              # total generator threads (otf_gen_tables total_streams)


def windowed_fits(cfg, smem_limit: int | None = None) -> tuple[bool, str]:
    """Is this config inside the windowed engine's limits (otf_engine_fits) and, when
    smem_limit is given, does its per-CTA shared memory fit the device?  Returns
    (fits, reason); scenarios that do not fit run on the exact engine."""
    L = _lib.lib()
    low = lower_any(cfg)
    c = low.cfg
    sc = _lib.Scenario()
    sc.n_clients, sc.n_workers, sc.n_seq, sc.n_ranks = c.clients, c.workers, len(low.seq_ids), low.n_ranks
    sc.max_nseg = max(low.counts)
    sc.latency, sc.horizon = float(c.client.latency_s), float(c.horizon_s)
    if not L.otf_engine_fits(_lib.ENGINE_WINDOWED, ctypes.byref(sc)):
        return False, (f"clients={sc.n_clients} workers={sc.n_workers} sequences={sc.n_seq} ranks={sc.n_ranks} "
                       f"segments/sequence={sc.max_nseg} latency={sc.latency}")
    if smem_limit is not None:
        smem = int(L.otf_shared_bytes(_lib.ENGINE_WINDOWED, sc.n_clients, sc.n_workers, sc.n_seq, sc.n_ranks,
                                      sc.max_nseg))
        if smem > smem_limit:
            return False, f"{smem} B of shared memory per scenario > {smem_limit} B"
    return True, ""


def _default_caps(low: Lowered) -> tuple[int, int, int, int]:
    cfg = low.cfg
    per_client = cfg.horizon_s / max(min(low.seq_segdur), 1e-3)
    req = int(cfg.clients * per_client * 1.25) + 256
    return req, req + cfg.clients, req, 2 * req + 64


def default_tail_caps(low: Lowered) -> tuple[int, int, int, int]:
    """Summary-tail capacities: nonzero request latencies, closed sessions, stalled
    sessions (the summary pass's gather), startup delays.

    Only requests that wait on a transcode have a nonzero latency (storage and
    cache hits answer at the arrival instant, server.py:61-78), so variants with
    every rank stored keep none and cache-less ones keep all; the rest are
    sized at a quarter of the expected requests.  A session lasts at least its
    sequence's duration unless the horizon cuts it, which bounds the sessions.
    A tail that overflows is counted exactly and the scenario re-run with it."""
    cfg = low.cfg
    req = _default_caps(low)[0]
    if len(low.stored) >= low.n_ranks:
        frac = 0.0
    elif not low.cache_enabled:
        frac = 1.0
    else:
        frac = 0.25
    sessions = cfg.clients * (int(cfg.horizon_s / max(min(low.seq_dur), 1e-3)) + 2)
    stalled = sessions if not low.cache_enabled else sessions // 4
    return int(req * frac) + 64, int(sessions) + 64, int(stalled) + 64, int(sessions) + 64


def _eps_len(low: Lowered) -> int:
    cfg = low.cfg
    rho = cfg.per_rank_rho or {r: cfg.rho for r, _ in cfg.ladder}
    min_dur = min(min(low.seq_segdur[i], low.seq_dur[i] - (low.counts[i] - 1) * low.seq_segdur[i])
                  for i in range(len(low.seq_ids)))
    floor = max(1.0 - 8.0 * cfg.noise_rel_std, 0.05)
    min_svc = max(min(rho.values()) * min_dur * floor, 1e-6)
    return int(min(cfg.horizon_s / min_svc + 64, 1 << 26))


_EPS_MEMO: dict = {}
_MAN_MEMO: dict = {}


def _manifest_bytes(low: Lowered, ladder, key) -> list[int]:
    """len(json.dumps(manifest_for(seq), sort_keys=True)) per sequence (server.py:58-59)."""
    man = _MAN_MEMO.get(key)
    if man is None:
        man = []
        for sid, dur, segdur, cnt in zip(low.seq_ids, low.seq_dur, low.seq_segdur, low.counts):
            m = {"sequence": sid, "duration_s": dur, "segment_duration_s": segdur, "segment_count": cnt,
                 "representations": [{"rank": r, "bitrate_bps": b} for r, b in ladder],
                 "url_template": URL_TEMPLATE}
            man.append(len(json.dumps(m, sort_keys=True).encode("utf-8")))
        if len(_MAN_MEMO) > 4096:
            _MAN_MEMO.clear()
        _MAN_MEMO[key] = man
    return man


def _eps_len_memo(low: Lowered) -> int:
    cfg = low.cfg
    key = (cfg.horizon_s, cfg.noise_rel_std, cfg.rho, tuple(sorted((cfg.per_rank_rho or {}).items())),
           tuple(cfg.ladder[i][0] for i in range(len(cfg.ladder))), tuple(low.seq_segdur), tuple(low.seq_dur))
    v = _EPS_MEMO.get(key)
    if v is None:
        v = _EPS_MEMO[key] = _eps_len(low)
    return v


def build_inputs(configs, engine: int = _lib.ENGINE_WINDOWED, mode: int = _lib.MODE_RECORDS,
                 caps=None, eps_scale: float = 1, threads: int | None = None, pin: bool = False,
                 tail_caps=None, list_caps=None) -> BatchInputs:
    """Lower a list of ExperimentConfigs into one device batch (host arrays; page-locked if pin)."""
    L = _lib.lib()
    threads = threads or os.cpu_count() or 1
    lows = [lower_any(c) for c in configs]
    P = _Pools(threads)
    scen = (_lib.Scenario * max(1, len(lows)))()
    tables = []
    scratch_off = 0
    cap_arr = np.zeros((len(lows), 4), dtype=np.int64)
    rec_off = np.zeros((len(lows), 4), dtype=np.int64)
    totals = [0, 0, 0, 0]
    input_bytes = 0
    shared_bytes = 0
    smem_per: list[int] = []
    tcap_arr = np.zeros((len(lows), 4), dtype=np.int64)
    ttot = [0, 0, 0]

    # -- device-generated tables first (the pool's device-only prefix) --
    jobs: list = []
    streams = 0

    def add_job(**kw) -> None:
        nonlocal streams
        first = (streams + _lib.GEN_ALIGN - 1) // _lib.GEN_ALIGN * _lib.GEN_ALIGN
        jobs.append(_lib.GenJob(first_stream=first, **kw))
        streams = first + kw["n_streams"]

    # traces: one table per (seed, netem), long enough for the largest N
    trace_groups: dict = {}
    for low in lows:
        if low.cfg.netem.trace_dir:
            continue                                   # CSV traces: per-client host tables below
        key = (low.cfg.seed, _netem_key(low.cfg.netem))
        prev = trace_groups.get(key, (0, low.cfg.netem))[0]
        trace_groups[key] = (max(prev, low.cfg.clients), low.cfg.netem)
    trace_tab = {}
    for key, (nmax, ne) in trace_groups.items():
        ts, period, grid = _trace_grid(ne.trace_duration_s, ne.step_s)
        n = len(ts)
        decay = math.exp(-ne.theta_per_s * ne.step_s)
        trace_tab[key] = dict(n=n, period=period, grid=grid, ts=ts, values=P.device("f64", nmax * n),
                              pbits=P.device("f64", nmax), nmax=nmax,
                              job=dict(kind=_lib.GEN_TRACE, n=n, n_streams=nmax, seed=key[0], period=period,
                                       mu=math.log(ne.median_bps), sigma=ne.sigma, decay=decay,
                                       spread=ne.sigma * math.sqrt(1.0 - decay * decay),
                                       floor_bps=ne.floor_bps, cap_bps=ne.cap_bps))
        input_bytes += 8 * (nmax * n + nmax + n)

    # worker noise: one table per (seed, noise), longest draw count
    eps_groups: dict = {}
    for low in lows:
        key = (low.cfg.seed, low.cfg.noise_rel_std)
        k, e = eps_groups.get(key, (0, 0))
        eps_groups[key] = (max(k, low.cfg.workers), max(e, max(1, int(_eps_len_memo(low) * eps_scale))))
    eps_tab = {}
    for (seed, noise), (kmax, elen) in eps_groups.items():
        if noise > 0:
            off = P.device("f64", kmax * elen)
            add_job(kind=_lib.GEN_NOISE, n=elen, n_streams=kmax, seed=seed, off_out=off, scale=noise)
            eps_tab[(seed, noise)] = (off, elen)

    # arrivals: one table per (seed, N, rate)
    arr_tab = {}
    for low in lows:
        akey = (low.cfg.seed, low.cfg.clients, low.cfg.arrival_rate_per_s)
        if akey not in arr_tab:
            off = P.device("f64", low.cfg.clients)
            add_job(kind=_lib.GEN_ARRIVALS, n=low.cfg.clients, n_streams=1, seed=low.cfg.seed, off_out=off,
                    scale=1.0 / low.cfg.arrival_rate_per_s)
            arr_tab[akey] = off
            input_bytes += 8 * low.cfg.clients

    # host parts from here on
    for (seed, noise), (kmax, elen) in eps_groups.items():
        if noise <= 0:
            eps_tab[(seed, noise)] = (P.add("f64", np.zeros((kmax, 1))), 1)
    for key, tt in trace_tab.items():
        tt["starts"] = P.add("f64", np.asarray(tt["ts"], dtype=np.float64))
        add_job(off_out=tt["values"], off_pbits=tt["pbits"], off_starts=tt["starts"], **tt["job"])

    cat_ids: dict = {}
    cat_groups: dict = {}
    for si, low in enumerate(lows):
        cfg = low.cfg
        N, K = cfg.clients, cfg.workers
        n_seq, n_ranks = len(low.seq_ids), low.n_ranks
        # the catalog tables: once per lowering (configs lowered from one memo entry share
        # seq_ids by identity; every Lowered of this call is alive, so ids are unique)
        gkey = (id(low.seq_ids), cfg.popularity, cfg.zipf_exponent)
        g = cat_groups.get(gkey)
        if g is None:
            max_nseg = max(low.counts)
            ladder = sorted(cfg.ladder)
            cat_key = cat_ids.setdefault(low.cat_key, len(cat_ids))   # small ids: the catalog tuples hash once
            ids_key = cat_ids.setdefault(low.cat_key[2], len(cat_ids))
            ladder_key = cat_ids.setdefault(low.cat_key[5], len(cat_ids))
            o_bitrates = P.add("i64", [b for _, b in ladder], key=("bitrates", ladder_key))
            if ("i64", ("keys", ids_key)) not in P.memo:
                keys = [int.from_bytes(hashlib.sha256(s.encode("utf-8")).digest()[:8], "big") for s in low.seq_ids]
                P.add("i64", np.array(keys, dtype=np.uint64).view(np.int64), key=("keys", ids_key))
            o_keys = P.memo[("i64", ("keys", ids_key))]
            o_seqdur = P.add("f64", low.seq_dur, key=("seqdur", cat_key))
            o_segdur = P.add("f64", low.seq_segdur, key=("segdur", cat_key))
            o_counts = P.add("i32", low.counts, key=("counts", cat_key))
            if ("i64", ("sizes", cat_key)) not in P.memo:
                o_sizes = P.reserve("i64", n_seq * n_ranks * max_nseg, key=("sizes", cat_key))
                t = _lib.SizeTable()
                t.n_seq, t.n_ranks, t.max_nseg = n_seq, n_ranks, max_nseg
                t.seed, t.size_jitter = cfg.seed, cfg.size_jitter
                t.off_out, t.off_keys, t.off_bitrates = o_sizes, o_keys, o_bitrates
                t.off_seqdur, t.off_segdur, t.off_segcount = o_seqdur, o_segdur, o_counts
                tables.append(t)
                input_bytes += 8 * n_seq * n_ranks * max_nseg
            o_sizes = P.memo[("i64", ("sizes", cat_key))]
            mkey = ("manifest", cat_ids.setdefault(low.cat_key[2:], len(cat_ids)))   # not seed-dependent
            if ("i64", mkey) not in P.memo:
                P.add("i64", _manifest_bytes(low, ladder, low.cat_key[2:]), key=mkey)
            o_man = P.memo[("i64", mkey)]
            rho_map = cfg.per_rank_rho or {r: cfg.rho for r, _ in ladder}
            o_rho = P.add("f64", [float(rho_map[r]) for r, _ in ladder], key=("rho", tuple(sorted(rho_map.items()))))
            pop = 1 if cfg.popularity == "zipf" else 0
            zkey = ("zipf", n_seq, pop, cfg.zipf_exponent)
            o_zipf = P.memo.get(("f64", zkey))
            if o_zipf is None:
                o_zipf = P.add("f64", zipf_cdf(n_seq, cfg.zipf_exponent) if pop else np.zeros(n_seq), key=zkey)
            g = cat_groups[gkey] = (o_bitrates, o_seqdur, o_segdur, o_counts, o_sizes, o_man, o_rho, o_zipf,
                                    pop, max_nseg)
        o_bitrates, o_seqdur, o_segdur, o_counts, o_sizes, o_man, o_rho, o_zipf, pop, max_nseg = g
        o_arr = arr_tab[(cfg.seed, N, cfg.arrival_rate_per_s)]
        if cfg.netem.trace_dir:                        # orchestrator.py:243-253
            tdir = cfg.netem.trace_dir
            files = sorted(os.path.join(tdir, f) for f in os.listdir(tdir) if f.endswith(".csv"))
            if not files:
                raise ConfigError(f"no trace CSVs in {tdir}")
            order = _gen([cfg.seed, 2]).permutation(len(files))
            ti, tf = [], []
            for c in range(N):
                f = files[order[c % len(files)]]
                if ("f64", ("csv", f)) not in P.memo:
                    st_, val_, per_, pb_ = load_trace_csv(f)
                    grid_ = float(st_[1] - st_[0]) if len(st_) > 1 else 0.0
                    if not (grid_ > 0 and all(x == float(i) * grid_ for i, x in enumerate(st_))):
                        grid_ = 0.0
                    o_st = P.add("f64", st_, key=("csv", f))
                    o_val = P.add("f64", val_, key=("csvv", f))
                    P.memo[("meta", f)] = (o_st, o_val, len(st_), per_, pb_, grid_)
                    input_bytes += 16 * len(st_)
                o_st, o_val, n_, per_, pb_, grid_ = P.memo[("meta", f)]
                ti += [o_st, o_val, n_]
                tf += [per_, pb_, grid_]
            tt = dict(n=0, period=0.0, grid=0.0, starts=0, values=0, pbits=0,
                      tr_i=P.add("i64", ti), tr_f=P.add("f64", tf))
        else:
            tt = trace_tab[(cfg.seed, _netem_key(cfg.netem))]
        o_eps, eps_stride = eps_tab[(cfg.seed, cfg.noise_rel_std)]

        sc = scen[si]
        sc.n_clients, sc.n_workers, sc.n_seq, sc.n_ranks = N, K, n_seq, n_ranks
        sc.max_nseg, sc.n_samples = max_nseg, tt["n"]
        sc.cache_enabled, sc.spec_enabled = int(low.cache_enabled), int(low.spec_enabled)
        sc.popularity = pop
        sc.stored_mask = sum(1 << r for r in low.stored)
        sc.cache_capacity = int(cfg.cache_capacity_bytes)
        sc.seed = cfg.seed
        sc.horizon = float(cfg.horizon_s)
        sc.latency = float(cfg.client.latency_s)
        b = cfg.client.buffer
        sc.target, sc.safe, sc.panic, sc.resume, sc.startup = b.target_s, b.safe_s, b.panic_s, b.resume_s, b.startup_s
        sc.alpha, sc.headroom = float(cfg.client.ewma_alpha), float(cfg.client.headroom)
        sc.noise = float(cfg.noise_rel_std)
        sc.period = tt["period"]
        sc.grid_step = tt["grid"]
        sc.queue_bound = int(cfg.queue_bound)
        sc.retries = int(cfg.client.retries)
        sc.retry_backoff = float(cfg.client.retry_backoff_s)
        sc.demand_priority = int(bool(cfg.demand_priority))
        sc.off_tr_i = tt.get("tr_i", -1)
        sc.off_tr_f = tt.get("tr_f", -1)
        sc.off_sizes, sc.off_bitrates, sc.off_manifest, sc.off_segcount = o_sizes, o_bitrates, o_man, o_counts
        sc.off_seqdur, sc.off_segdur, sc.off_rho, sc.off_zipf = o_seqdur, o_segdur, o_rho, o_zipf
        sc.off_starts, sc.off_values, sc.off_pbits = tt["starts"], tt["values"], tt["pbits"]
        sc.off_arrivals = o_arr
        sc.off_eps, sc.eps_stride = o_eps, eps_stride
        sc.scratch_off = scratch_off
        lc = int(list_caps[si]) if list_caps is not None and list_caps[si] else 0
        scratch, smem = _engine_bytes(engine, N, K, n_seq, n_ranks, max_nseg, lc)
        scratch_off += scratch
        sc.list_cap = lc
        smem_per.append(smem)
        shared_bytes = max(shared_bytes, smem)
        scratch_off = (scratch_off + 255) & ~255
        tc = tail_caps[si] if tail_caps is not None and tail_caps[si] is not None else default_tail_caps(low)
        tcap_arr[si] = tc
        sc.lat_off, sc.lat_cap = int(ttot[0]), int(tc[0])
        sc.ses_off, sc.ses_cap, sc.stl_cap = int(ttot[1]), int(tc[1]), int(tc[2])
        sc.sup_off, sc.sup_cap = int(ttot[2]), int(tc[3])
        ttot[0] += int(tc[0])
        ttot[1] += int(tc[1]) + 2 * int(tc[2])         # records + the summary pass's gather and sort
        ttot[2] += int(tc[3])
        if mode == _lib.MODE_RECORDS:
            c = caps[si] if caps is not None else _default_caps(low)
            cap_arr[si] = c
            for k in range(4):
                rec_off[si, k] = totals[k]
                totals[k] += int(c[k])
            sc.req_off, sc.req_cap = int(rec_off[si, 0]), int(c[0])
            sc.sess_off, sc.sess_cap = int(rec_off[si, 1]), int(c[1])
            sc.seg_off, sc.seg_cap = int(rec_off[si, 2]), int(c[2])
            sc.job_off, sc.job_cap = int(rec_off[si, 3]), int(c[3])

    return BatchInputs(
        lowered=lows, scenarios=scen, size_tables=(_lib.SizeTable * max(1, len(tables)))(*tables),
        f64=P.concat("f64", pin), i64=P.concat("i64", pin), i32=P.concat("i32", pin), pinned=pin,
        scratch_bytes=max(scratch_off, 256), caps=cap_arr, rec_offsets=rec_off, rec_totals=totals,
        engine=engine, mode=mode, input_bytes=input_bytes, shared_bytes=shared_bytes, smem_per=smem_per,
        tail_caps=tcap_arr, tail_totals=tuple(ttot), f64_dev=P.dev["f64"],
        gen_jobs=(_lib.GenJob * max(1, len(jobs)))(*jobs), gen_streams=streams)


def n_size_tables(inp: BatchInputs) -> int:
    return sum(1 for t in inp.size_tables if t.n_seq > 0)


def n_gen_jobs(inp: BatchInputs) -> int:
    return inp.gen_streams and len(inp.gen_jobs) or 0


def host_generate(inp: BatchInputs, threads: int | None = None) -> np.ndarray:
    """The device-only f64 prefix as the HOST generators (csrc/otf_hostgen.cu) make it:
    the same jobs otf_gen_tables runs on the GPU, for tests (bit-for-bit equal)."""
    L = _lib.lib()
    threads = threads or os.cpu_count() or 1
    out = np.zeros(max(1, inp.f64_dev), dtype=np.float64)
    host = inp.f64
    dp = lambda a, off: a[off:].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    for j in inp.gen_jobs[:n_gen_jobs(inp)]:
        if j.kind == _lib.GEN_TRACE:
            starts = np.ascontiguousarray(host[j.off_starts - inp.f64_dev:j.off_starts - inp.f64_dev + j.n])
            _lib.check(L.otf_gen_traces(j.seed, j.n_streams, j.n, dp(starts, 0), j.period, j.mu, j.sigma, j.decay,
                                        j.spread, j.floor_bps, j.cap_bps, dp(out, j.off_out), dp(out, j.off_pbits),
                                        threads), "otf_gen_traces")
        elif j.kind == _lib.GEN_ARRIVALS:
            _lib.check(L.otf_gen_arrivals(j.seed, j.n, j.scale, dp(out, j.off_out)), "otf_gen_arrivals")
        elif j.kind == _lib.GEN_NOISE:
            _lib.check(L.otf_gen_noise(j.seed, int(j.n_streams), j.scale, j.n, dp(out, j.off_out), threads),
                       "otf_gen_noise")
    return out[:inp.f64_dev]
