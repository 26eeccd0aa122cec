"""Shared parity helpers: load golden fixtures, compare SoA result dicts.

Discrete fields must match exactly; float fields are compared bit-exactly by
default (the engines follow the reference's operation order with FMA
contraction disabled) with an optional relative tolerance (north star:
<= 1e-6 relative for float times and QoE scores).
"""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

INT_FIELDS = ["req_id", "req_seq", "req_rep", "req_index", "req_path", "req_bytes",
              "sess_client", "sess_seq", "sess_stalls", "sess_flags",
              "seg_session", "seg_index", "seg_rep",
              "job_seq", "job_rep", "job_index", "job_origin", "job_outcome"]
FLOAT_FIELDS = ["req_arrival", "req_response", "sess_start", "sess_end", "sess_stall_time",
                "sess_startup", "seg_start", "seg_end", "job_enq", "job_start", "job_fin"]


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN_DIR) if f.endswith(".npz"))


def load_golden(name: str):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    meta = json.loads(bytes(z["meta"]).decode("utf-8"))
    return arrays, meta


def normalise_segments(res: dict) -> dict:
    """Order segments by session (stable): the reference stores them per session."""
    out = dict(res)
    order = np.argsort(res["seg_session"], kind="stable")
    for k in ("seg_session", "seg_index", "seg_rep", "seg_start", "seg_end"):
        out[k] = np.asarray(res[k])[order]
    return out


def compare(got: dict, want: dict, rtol: float = 0.0) -> list[str]:
    """Return a list of human-readable mismatches (empty == parity)."""
    got = normalise_segments(got)
    want = normalise_segments(want)
    errs = []
    for k in INT_FIELDS:
        a, b = np.asarray(got[k]), np.asarray(want[k])
        if a.shape != b.shape:
            errs.append(f"{k}: length {a.shape} != {b.shape}")
            continue
        bad = np.nonzero(a.astype(np.int64) != b.astype(np.int64))[0]
        if bad.size:
            i = bad[0]
            errs.append(f"{k}: {bad.size} mismatches, first at {i}: {a[i]} != {b[i]}")
    for k in FLOAT_FIELDS:
        a, b = np.asarray(got[k], dtype=np.float64), np.asarray(want[k], dtype=np.float64)
        if a.shape != b.shape:
            errs.append(f"{k}: length {a.shape} != {b.shape}")
            continue
        nan_a, nan_b = np.isnan(a), np.isnan(b)
        if (nan_a != nan_b).any():
            i = np.nonzero(nan_a != nan_b)[0][0]
            errs.append(f"{k}: None/NaN pattern differs at {i}: {a[i]} vs {b[i]}")
            continue
        m = ~nan_a
        if rtol == 0.0:
            bad = np.nonzero(a[m].view(np.int64) != b[m].view(np.int64))[0]
        else:
            bad = np.nonzero(np.abs(a[m] - b[m]) > rtol * np.maximum(np.abs(b[m]), 1e-300))[0]
        if bad.size:
            i = bad[0]
            errs.append(f"{k}: {bad.size} mismatches, first at {i}: {a[m][i]!r} != {b[m][i]!r}")
    return errs


def compare_stats(got: dict, want: dict) -> list[str]:
    errs = []
    for k in sorted(set(got) | set(want)):
        if got.get(k) != want.get(k):
            errs.append(f"backend_stats[{k}]: {got.get(k)} != {want.get(k)}")
    return errs
