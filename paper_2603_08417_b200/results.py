"""Result objects with the reference's shape (server.py:31-44, client.py:149-187,
transcode.py:102-110, orchestrator.py:271-324) plus the metrics the reference
computes from them (metrics.py:52-162).

A ``ExperimentResult`` is built lazily from the engine's SoA arrays: the
``arrays`` dict is always available (numpy views, cheap), and the object
lists ``requests`` / ``sessions`` / ``jobs`` are materialised on first access.
"""

from __future__ import annotations

import csv
import hashlib
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["SegmentDescriptor", "RequestRecord", "SegmentRecord", "SessionReport", "TranscodeJob",
           "ExperimentResult", "fingerprint", "response_time_cdf", "stalls_per_session",
           "quality_proportions", "INSTANT_EPSILON_S", "SCHEMAS", "read_csv"]

INSTANT_EPSILON_S = 0.010
PATHS = ("storage", "cache", "waited_inflight", "transcoded", "error")
ORIGINS = ("demand", "speculative")
OUTCOMES = ("pending", "completed", "dropped", "failed")


@dataclass(frozen=True)
class SegmentDescriptor:
    sequence: str
    rep: int
    index: int
    duration: float
    size: int


@dataclass(frozen=True)
class RequestRecord:
    request_id: int
    sequence: str
    rep: int
    index: int
    arrival_s: float
    response_s: float
    path: str
    nbytes: int

    @property
    def latency_s(self) -> float:
        return self.response_s - self.arrival_s


@dataclass(frozen=True)
class SegmentRecord:
    index: int
    rep: int
    dl_start_s: float
    dl_end_s: float


@dataclass
class SessionReport:
    client_id: int
    sequence: str
    start_s: float
    end_s: float = 0.0
    stalls: int = 0
    stall_time_s: float = 0.0
    startup_delay_s: float | None = None
    segments: list[SegmentRecord] = field(default_factory=list)
    finished: bool = False
    aborted: bool = False

    @property
    def mean_rank(self) -> float:
        if not self.segments:
            return 0.0
        return sum(s.rep for s in self.segments) / len(self.segments)


@dataclass
class TranscodeJob:
    target: SegmentDescriptor
    source_rank: int
    origin: str
    enqueued_at: float
    started_at: float | None = None
    finished_at: float | None = None
    outcome: str = "pending"


def fingerprint(config: dict) -> str:
    """Stable 12-hex digest of a JSON config (metrics.py:52-55)."""
    blob = json.dumps(config, sort_keys=True, separators=(",", ":")).encode("utf-8")
    return hashlib.sha256(blob).hexdigest()[:12]


@dataclass(frozen=True)
class CdfSummary:
    points: list
    instant_fraction: float


def response_time_cdf(records, epsilon_s: float = INSTANT_EPSILON_S) -> CdfSummary:
    """metrics.py:67-78"""
    if not records:
        raise ValueError("no request records")
    latencies = sorted(r.latency_s for r in records)
    n = len(latencies)
    points = []
    for i, lat in enumerate(latencies):
        if i + 1 < n and latencies[i + 1] == lat:
            continue
        points.append((lat, (i + 1) / n))
    instant = sum(1 for lat in latencies if lat < epsilon_s) / n
    return CdfSummary(points, instant)


@dataclass(frozen=True)
class StallSummary:
    counts: list
    mean: float
    total_stall_time_s: float


def stalls_per_session(sessions) -> StallSummary:
    """metrics.py:88-92"""
    if not sessions:
        raise ValueError("no sessions")
    counts = [s.stalls for s in sessions]
    # The reference's stall times are np.float64 once a session has stalled
    # (they accumulate loop.now() differences), which knocks CPython's sum()
    # off its compensated float path: the total is a plain left-to-right sum.
    total = 0.0
    for s in sessions:
        total += s.stall_time_s
    return StallSummary(counts, sum(counts) / len(counts), total)


@dataclass(frozen=True)
class QualitySummary:
    fractions: dict
    mean_rank: float
    segment_count: int


def quality_proportions(sessions, ladder_size: int, sequence: str | None = None) -> QualitySummary:
    """metrics.py:102-116"""
    counts = {rank: 0 for rank in range(1, ladder_size + 1)}
    total = 0
    for session in sessions:
        if sequence is not None and session.sequence != sequence:
            continue
        for seg in session.segments:
            counts[seg.rep] += 1
            total += 1
    if total == 0:
        raise ValueError("no downloaded segments to aggregate")
    fractions = {rank: c / total for rank, c in counts.items()}
    mean_rank = sum(rank * frac for rank, frac in fractions.items())
    return QualitySummary(fractions, mean_rank, total)


SCHEMAS = {  # metrics.py:40-49
    "requests": ("requests.v1", ["request_id", "seq", "rep", "index", "arrival_s", "response_s", "path", "bytes"]),
    "sessions": ("sessions.v1", ["client_id", "seq", "variant", "stalls", "stall_time_s", "startup_delay_s"]),
    "segments": ("segments.v1", ["client_id", "seq", "index", "rep", "dl_start_s", "dl_end_s"]),
    "jobs": ("jobs.v1", ["seq", "rep", "index", "origin", "enqueued_s", "started_s", "finished_s", "outcome"]),
}


def _fmt(x) -> str:
    if x is None:
        return ""
    if isinstance(x, float):
        return f"{x:.6f}"
    return str(x)


def _write(path, schema_key: str, config_hex: str, rows) -> None:
    name, columns = SCHEMAS[schema_key]
    with open(path, "w", newline="", encoding="utf-8") as fh:
        fh.write(f"# schema={name} config={config_hex}\n")
        w = csv.writer(fh)
        w.writerow(columns)
        for row in rows:
            w.writerow([_fmt(v) for v in row])


def read_csv(path, schema_key: str):
    """Load a bundle CSV written by `_write` (the reader of metrics.py:165-181):
    (header tags, rows as dicts).  The `# schema=... config=...` tag line and the
    column row must match the writer's current schema, else ValueError."""
    want_name, want_cols = SCHEMAS[schema_key]
    with open(path, newline="", encoding="utf-8") as fh:
        rows = csv.reader(fh)
        tag = next(rows, [""])
        tag_line = ",".join(tag).strip()
        if not tag_line.startswith("# schema="):
            raise ValueError(f"{path}: missing schema header")
        tags = {}
        for item in tag_line[1:].split():
            key, _, val = item.partition("=")
            tags[key] = val
        if tags.get("schema") != want_name:
            raise ValueError(f"{path}: schema {tags.get('schema')!r} != expected {want_name!r}")
        cols = next(rows, None)
        if cols != want_cols:
            raise ValueError(f"{path}: columns {cols} != expected {want_cols}")
        return tags, [dict(zip(cols, r)) for r in rows]


def _opt(x: float):
    return None if np.isnan(x) else float(x)


class ExperimentResult:
    """orchestrator.py:271-324, backed by the engine's SoA arrays."""

    def __init__(self, config, arrays: dict, stats: np.ndarray, seq_ids: list[str], sizes=None,
                 seq_dur=None, seq_segdur=None, qoe: dict | None = None, status: int = 0, counts=None):
        self.config = config
        self.arrays = arrays
        self.stats_raw = stats
        self.seq_ids = seq_ids
        self._qoe = qoe                                # dict, or a raw otf_qoe row parsed on first use
        self.qoe_row = None if isinstance(qoe, dict) or qoe is None else np.asarray(qoe)
        self.counts = None if counts is None else np.asarray(counts)   # requests, sessions, segments, jobs
        self.status = status
        self._sizes = sizes
        self._seq_dur = seq_dur
        self._seq_segdur = seq_segdur
        self._requests = self._sessions = self._jobs = None
        self._fingerprint = self._bstats = None

    # derived fields are computed on first use: a 1,024-scenario sweep returns 1,024 results
    @property
    def fingerprint(self) -> str:
        if self._fingerprint is None:
            self._fingerprint = fingerprint(self.config.to_dict())
        return self._fingerprint

    @property
    def backend_stats(self) -> dict:
        if self._bstats is None:
            self._bstats = self._backend_stats()
        return self._bstats

    @property
    def qoe(self):
        if self._qoe is not None and not isinstance(self._qoe, dict):
            from .engine import parse_qoe
            self._qoe = parse_qoe(self._qoe)
        return self._qoe

    def _backend_stats(self) -> dict:
        st = self.stats_raw
        skipped = {r: int(st[_lib.ST["skip0"] + i]) for i, r in enumerate(_lib.SKIP_REASONS)
                   if st[_lib.ST["skip0"] + i]}
        out = {"jobs_total": int(st[0]), "jobs_demand": int(st[1]), "jobs_speculative": int(st[2]),
               "wasted_avoided": int(st[3]), "speculation_enqueued": int(st[4]),
               "speculation_skipped": skipped}
        if self.config.policy().cache_enabled:
            out["cache"] = {k: int(st[_lib.ST[k]]) for k in
                            ("capacity_bytes", "current_bytes", "entries", "hits", "misses", "evictions",
                             "rejected")}
        return out

    def _need_records(self, what: str) -> None:
        if not self.arrays:
            raise _lib.OtfError(f"ExperimentResult.{what} needs per-request records: this result comes from a "
                                f"histogram-mode run; use run_batch(..., mode='records') (summary() works in both)")

    @property
    def requests(self) -> list[RequestRecord]:
        self._need_records("requests")
        if self._requests is None:
            a = self.arrays
            ids = self.seq_ids
            self._requests = [
                RequestRecord(int(i), ids[s], int(r), int(x), float(t0), float(t1), PATHS[p], int(nb))
                for i, s, r, x, t0, t1, p, nb in zip(a["req_id"], a["req_seq"], a["req_rep"], a["req_index"],
                                                     a["req_arrival"], a["req_response"], a["req_path"],
                                                     a["req_bytes"])]
        return self._requests

    @property
    def sessions(self) -> list[SessionReport]:
        self._need_records("sessions")
        if self._sessions is None:
            a = self.arrays
            ids = self.seq_ids
            out = [SessionReport(int(c), ids[s], float(t0), float(t1), int(n), float(st), _opt(su),
                                 [], bool(f & 1), bool(f & 2))
                   for c, s, t0, t1, n, st, su, f in zip(a["sess_client"], a["sess_seq"], a["sess_start"],
                                                         a["sess_end"], a["sess_stalls"], a["sess_stall_time"],
                                                         a["sess_startup"], a["sess_flags"])]
            for sess, idx, rep, t0, t1 in zip(a["seg_session"], a["seg_index"], a["seg_rep"], a["seg_start"],
                                              a["seg_end"]):
                out[sess].segments.append(SegmentRecord(int(idx), int(rep), float(t0), float(t1)))
            self._sessions = out
        return self._sessions

    @property
    def jobs(self) -> list[TranscodeJob]:
        self._need_records("jobs")
        if self._jobs is None:
            a = self.arrays
            ids = self.seq_ids
            top = len(self.config.ladder)
            out = []
            for s, r, x, o, oc, te, ts, tf in zip(a["job_seq"], a["job_rep"], a["job_index"], a["job_origin"],
                                                  a["job_outcome"], a["job_enq"], a["job_start"], a["job_fin"]):
                dur = min(self._seq_segdur[s], self._seq_dur[s] - x * self._seq_segdur[s])
                desc = SegmentDescriptor(ids[s], int(r), int(x), dur, int(self._sizes[s, r - 1, x]))
                out.append(TranscodeJob(desc, top, ORIGINS[o], float(te), _opt(ts), _opt(tf), OUTCOMES[oc]))
            self._jobs = out
        return self._jobs

    def summary(self) -> dict:
        """orchestrator.py:280-309.  Records mode: from the records, as the reference.
        Histogram mode: from the device's QoE block, field for field the same values
        (otf_qoe in include/otfgpu.h lists how each one is formed)."""
        if not self.arrays:
            return self._summary_from_qoe()
        ladder_size = max(rank for rank, _ in self.config.ladder)
        n_req = len(self.arrays["req_id"])
        out = {
            "fingerprint": self.fingerprint,
            "variant": self.config.variant,
            "clients": self.config.clients,
            "workers": self.config.workers,
            "segment_duration_s": self.config.segment_duration_s,
            "requests": n_req,
            "sessions": len(self.arrays["sess_client"]),
            "jobs": len(self.arrays["job_seq"]),
            "backend": self.backend_stats,
        }
        if n_req:
            cdf = response_time_cdf(self.requests)
            out["instant_fraction"] = cdf.instant_fraction
            lat = sorted(r.latency_s for r in self.requests)
            out["latency_p50_s"] = lat[len(lat) // 2]
            out["latency_p99_s"] = lat[min(len(lat) - 1, int(0.99 * len(lat)))]
        if len(self.arrays["sess_client"]):
            stalls = stalls_per_session(self.sessions)
            out["stalls_mean"] = stalls.mean
            out["stall_time_total_s"] = stalls.total_stall_time_s
            try:
                quality = quality_proportions(self.sessions, ladder_size)
                out["quality_fractions"] = {str(k): v for k, v in quality.fractions.items()}
                out["mean_rank"] = quality.mean_rank
            except ValueError:
                pass
        return out

    def _summary_from_qoe(self) -> dict:
        q = self.qoe
        if q is None:
            raise _lib.OtfError("no QoE block in this result")
        ladder_size = max(rank for rank, _ in self.config.ladder)
        n_req, n_sess = int(q["n_requests"]), int(q["n_sessions"])
        jobs = int(self.counts[3]) if self.counts is not None else int(self.stats_raw[_lib.ST["jobs_total"]])
        out = {
            "fingerprint": self.fingerprint,
            "variant": self.config.variant,
            "clients": self.config.clients,
            "workers": self.config.workers,
            "segment_duration_s": self.config.segment_duration_s,
            "requests": n_req,
            "sessions": n_sess,
            "jobs": jobs,
            "backend": self.backend_stats,
        }
        if n_req:
            if not q["summary_flags"] & _lib.Q_ORDER_STATS:
                raise _lib.OtfError("the summary pass did not run for this scenario (status %#x)" % self.status)
            out["instant_fraction"] = q["lat_hist"][0] / n_req          # metrics.py:77
            out["latency_p50_s"] = q["latency_p50"]
            out["latency_p99_s"] = q["latency_p99"]
        if n_sess:
            out["stalls_mean"] = int(q["n_stalls"]) / n_sess              # metrics.py:91
            out["stall_time_total_s"] = q["stall_time_sum"]
            total = int(q["n_segments"])
            if total:
                if ladder_size >= _lib.RANK_BINS or q["summary_flags"] & _lib.Q_RANKS_CAPPED:
                    raise _lib.OtfError(f"quality fractions need ranks < {_lib.RANK_BINS} in histogram mode")
                fractions = {rank: int(q["rank_count"][rank]) / total for rank in range(1, ladder_size + 1)}
                out["quality_fractions"] = {str(k): v for k, v in fractions.items()}
                out["mean_rank"] = sum(rank * frac for rank, frac in fractions.items())   # metrics.py:115
        return out

    def write(self, outdir) -> None:
        """orchestrator.py:311-324 + metrics.py:140-162"""
        os.makedirs(outdir, exist_ok=True)
        fp = self.fingerprint
        _write(os.path.join(outdir, "requests.csv"), "requests", fp,
               ((r.request_id, r.sequence, r.rep, r.index, r.arrival_s, r.response_s, r.path, r.nbytes)
                for r in self.requests))
        _write(os.path.join(outdir, "sessions.csv"), "sessions", fp,
               ((s.client_id, s.sequence, self.config.variant, s.stalls, s.stall_time_s, s.startup_delay_s)
                for s in self.sessions))
        _write(os.path.join(outdir, "segments.csv"), "segments", fp,
               ((s.client_id, s.sequence, g.index, g.rep, g.dl_start_s, g.dl_end_s)
                for s in self.sessions for g in s.segments))
        _write(os.path.join(outdir, "jobs.csv"), "jobs", fp,
               ((j.target.sequence, j.target.rep, j.target.index, j.origin, j.enqueued_at, j.started_at,
                 j.finished_at, j.outcome) for j in self.jobs))
        with open(os.path.join(outdir, "config.json"), "w", encoding="utf-8") as fh:
            json.dump({"fingerprint": fp, **self.config.to_dict()}, fh, indent=2, sort_keys=True)
            fh.write("\n")
        with open(os.path.join(outdir, "summary.json"), "w", encoding="utf-8") as fh:
            json.dump(self.summary(), fh, indent=2, sort_keys=True)
            fh.write("\n")
