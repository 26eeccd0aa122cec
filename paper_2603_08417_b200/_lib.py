"""ctypes binding of libotfgpu.so (include/otfgpu.h).

The library is built in-tree (``paper_2603_08417_b200/libotfgpu.so``) by
``build()`` / ``__graft_entry__.build()``.  There is no fallback: every
product entry point goes through this module and raises when the library or
a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_PATH = os.environ.get("OTFGPU_LIB_OVERRIDE") or os.path.join(HERE, "libotfgpu.so")   # override: tools/ experiments
ABI_VERSION = 3

_P = ctypes.POINTER
_vp = ctypes.c_void_p
_i32, _u32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double

# enums (values are part of the ABI)
PATH_STORAGE, PATH_CACHE, PATH_WAITED, PATH_TRANSCODED, PATH_ERROR = 0, 1, 2, 3, 4
ORIGIN_DEMAND, ORIGIN_SPECULATIVE = 0, 1
OUTCOME_PENDING, OUTCOME_COMPLETED, OUTCOME_DROPPED = 0, 1, 2
POP_UNIFORM, POP_ZIPF = 0, 1
ENGINE_EXACT, ENGINE_WINDOWED = 0, 1
MODE_HISTOGRAM, MODE_RECORDS = 0, 1
S_RECORD_OVERFLOW, S_EPS_OVERFLOW, S_INTERNAL, S_TIE, S_HUNG, S_UNFIT, S_TAIL_OVERFLOW, S_LIST_OVERFLOW = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40, 0x80)
Q_ORDER_STATS, Q_INEXACT_SUM, Q_RANKS_CAPPED = 0x1, 0x2, 0x4
BF_ENGINE_ONLY = 0x1
SM_COUNT_B200, SMEM_PER_SM = 148, 227 * 1024

ST_NSLOTS = 32
ST = dict(jobs_total=0, jobs_demand=1, jobs_speculative=2, wasted_avoided=3, speculation_enqueued=4,
          skip0=5, capacity_bytes=11, current_bytes=12, entries=13, hits=14, misses=15,
          evictions=16, rejected=17, status=18, hung=19, timer_pops=20, ready_callbacks=21, windows=22,
          cyc_scan=23, cyc_sort=24, cyc_server=25, cyc_clients=26, cyc_total=27)
SKIP_REASONS = ("disabled", "end-of-sequence", "stored", "cached", "in-flight", "overload")
LAT_BINS, STALL_BINS, RANK_BINS = 64, 32, 32


class Scenario(ctypes.Structure):
    _fields_ = [
        ("n_clients", _i32), ("n_workers", _i32), ("n_seq", _i32), ("n_ranks", _i32),
        ("max_nseg", _i32), ("n_samples", _i32), ("cache_enabled", _i32), ("spec_enabled", _i32),
        ("popularity", _i32), ("queue_bound", _i32), ("stored_mask", _u32), ("retries", _i32),
        ("cache_capacity", _i64), ("seed", _u64),
        ("horizon", _f64), ("latency", _f64),
        ("target", _f64), ("safe", _f64), ("panic", _f64), ("resume", _f64), ("startup", _f64),
        ("alpha", _f64), ("headroom", _f64), ("noise", _f64), ("period", _f64), ("grid_step", _f64), ("retry_backoff", _f64),
        ("demand_priority", _i32), ("list_cap", _i32), ("off_tr_i", _i64), ("off_tr_f", _i64),
        ("off_sizes", _i64), ("off_bitrates", _i64), ("off_manifest", _i64), ("off_segcount", _i64),
        ("off_seqdur", _i64), ("off_segdur", _i64), ("off_rho", _i64), ("off_zipf", _i64),
        ("off_starts", _i64), ("off_values", _i64), ("off_pbits", _i64), ("off_arrivals", _i64),
        ("off_eps", _i64), ("eps_stride", _i64), ("scratch_off", _i64),
        ("req_off", _i64), ("req_cap", _i64), ("sess_off", _i64), ("sess_cap", _i64),
        ("seg_off", _i64), ("seg_cap", _i64), ("job_off", _i64), ("job_cap", _i64),
        ("lat_off", _i64), ("lat_cap", _i64), ("ses_off", _i64), ("ses_cap", _i64), ("stl_cap", _i64),
        ("sup_off", _i64), ("sup_cap", _i64),
    ]


class Qoe(ctypes.Structure):
    _fields_ = [
        ("lat_hist", _i64 * LAT_BINS), ("path_count", _i64 * 8), ("stall_hist", _i64 * STALL_BINS),
        ("rank_count", _i64 * RANK_BINS),
        ("n_requests", _i64), ("n_sessions", _i64), ("n_segments", _i64), ("n_finished", _i64),
        ("n_started", _i64), ("n_stalls", _i64),
        ("latency_sum", _f64), ("stall_time_sum", _f64), ("startup_delay_sum", _f64),
        ("latency_p50", _f64), ("latency_p99", _f64),
        ("n_lat_tail", _i64), ("n_stall_tail", _i64), ("summary_flags", _i64),
    ]


SESS_ENT_BYTES = 24    # otf_sess_ent: reg_time f64, stall_time f64, sid i32, stalls u32


RECORD_FIELDS = [  # (name, numpy dtype) in otf_batch order
    ("req_id", "i8"), ("req_seq", "i4"), ("req_rep", "i4"), ("req_index", "i4"), ("req_path", "i4"),
    ("req_arrival", "f8"), ("req_response", "f8"), ("req_bytes", "i8"),
    ("sess_client", "i4"), ("sess_seq", "i4"), ("sess_stalls", "i4"), ("sess_flags", "i4"),
    ("sess_start", "f8"), ("sess_end", "f8"), ("sess_stall_time", "f8"), ("sess_startup", "f8"),
    ("seg_session", "i4"), ("seg_index", "i4"), ("seg_rep", "i4"), ("seg_start", "f8"), ("seg_end", "f8"),
    ("job_seq", "i4"), ("job_rep", "i4"), ("job_index", "i4"), ("job_origin", "i4"), ("job_outcome", "i4"),
    ("job_enq", "f8"), ("job_start", "f8"), ("job_fin", "f8"),
]


class Batch(ctypes.Structure):
    _fields_ = ([("n_scenarios", _i32), ("mode", _i32), ("scenarios", _vp), ("f64_pool", _vp),
                 ("i64_pool", _vp), ("i32_pool", _vp), ("scratch", _vp)]
                + [(n, _vp) for n, _ in RECORD_FIELDS]
                + [("counts", _vp), ("stats", _vp), ("qoe", _vp), ("status", _vp), ("order", _vp),
                   ("shared_bytes", _i64), ("engine_flags", _i32), ("concurrent", _i32),
                   ("tail_lat", _vp), ("tail_sess", _vp), ("tail_sup", _vp)])


class TraceJob(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_traces", _i64), ("n_samples", _i32), ("pad", _i32),
                ("starts", _vp), ("period", _f64), ("mu", _f64), ("sigma", _f64), ("decay", _f64),
                ("spread", _f64), ("floor_bps", _f64), ("cap_bps", _f64), ("values", _vp), ("pbits", _vp)]


GEN_TRACE, GEN_ARRIVALS, GEN_NOISE = 0, 1, 2
GEN_ALIGN = 128


class GenJob(ctypes.Structure):
    _fields_ = [("kind", _i32), ("n", _i32), ("n_streams", _i64), ("first_stream", _i64), ("seed", _u64),
                ("off_out", _i64), ("off_pbits", _i64), ("off_starts", _i64),
                ("period", _f64), ("mu", _f64), ("sigma", _f64), ("decay", _f64), ("spread", _f64),
                ("floor_bps", _f64), ("cap_bps", _f64), ("scale", _f64)]


class SizeTable(ctypes.Structure):
    _fields_ = [
        ("n_seq", _i32), ("n_ranks", _i32), ("max_nseg", _i32), ("pad", _i32),
        ("seed", _u64), ("size_jitter", _f64),
        ("off_out", _i64), ("off_keys", _i64), ("off_bitrates", _i64),
        ("off_seqdur", _i64), ("off_segdur", _i64), ("off_segcount", _i64),
    ]


EXPORTS = ("otf_version", "otf_last_error", "otf_sizeof_scenario", "otf_sizeof_batch", "otf_sizeof_qoe",
           "otf_scratch_bytes", "otf_shared_bytes", "otf_shared_bytes_cap", "otf_list_cap", "otf_engine_fits", "otf_build_traces", "otf_np_draws", "otf_gen_arrivals",
           "otf_gen_noise", "otf_gen_traces", "otf_gen_traces_multi", "otf_model_completion_time",
           "otf_model_select_quality", "otf_model_buffer_run", "otf_model_exact_sum", "otf_model_completion_times", "otf_gen_sizes", "otf_gen_tables",
           "otf_model_libm", "otf_model_libm_dev", "otf_run_batch", "otf_run_summary")
DRAW_STANDARD_NORMAL, DRAW_NORMAL, DRAW_EXPONENTIAL, DRAW_STANDARD_EXPONENTIAL = 0, 1, 2, 3


class OtfError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile libotfgpu.so for sm_100a in place (csrc/Makefile)."""
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h", "Makefile"))]
    srcs.append(os.path.join(os.path.dirname(HERE), "include", "otfgpu.h"))
    stale = not os.path.exists(LIB_PATH) or any(os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in srcs)
    if force or stale:
        subprocess.run(["make", "-s"] + (["-B"] if force else []) + ["-C", CSRC], check=True)
    return LIB_PATH


_lib = None


def lib():
    """Load libotfgpu.so (fails loudly if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OtfError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(LIB_PATH)
    L.otf_version.restype = ctypes.c_int
    L.otf_last_error.restype = ctypes.c_char_p
    for f in ("otf_sizeof_scenario", "otf_sizeof_batch", "otf_sizeof_qoe"):
        getattr(L, f).restype = ctypes.c_size_t
    L.otf_scratch_bytes.restype = _i64
    L.otf_scratch_bytes.argtypes = [_i32] * 6
    L.otf_engine_fits.restype = _i32
    L.otf_engine_fits.argtypes = [_i32, _P(Scenario)]
    L.otf_shared_bytes.restype = _i64
    L.otf_shared_bytes.argtypes = [_i32] * 6
    L.otf_shared_bytes_cap.restype = _i64
    L.otf_shared_bytes_cap.argtypes = [_i32] * 5
    L.otf_list_cap.restype = _i32
    L.otf_list_cap.argtypes = [_i32]
    L.otf_build_traces.restype = ctypes.c_int
    L.otf_build_traces.argtypes = [_i64, _i32, _P(_f64), _P(_f64), _f64, _f64, _f64, _f64, _f64, _f64, _f64,
                                   _P(_f64), _P(_f64), _i32]
    L.otf_np_draws.restype = ctypes.c_int
    L.otf_np_draws.argtypes = [_i32, _P(ctypes.c_uint64), _i32, _f64, _f64, _i64, _P(_f64)]
    L.otf_gen_arrivals.restype = ctypes.c_int
    L.otf_gen_arrivals.argtypes = [ctypes.c_uint64, _i64, _f64, _P(_f64)]
    L.otf_gen_noise.restype = ctypes.c_int
    L.otf_gen_noise.argtypes = [ctypes.c_uint64, _i32, _f64, _i64, _P(_f64), _i32]
    L.otf_gen_traces.restype = ctypes.c_int
    L.otf_gen_traces.argtypes = [ctypes.c_uint64, _i64, _i32, _P(_f64), _f64, _f64, _f64, _f64, _f64, _f64, _f64,
                                 _P(_f64), _P(_f64), _i32]
    L.otf_gen_traces_multi.restype = ctypes.c_int
    L.otf_gen_traces_multi.argtypes = [_i32, _vp, _i32]
    L.otf_model_completion_time.restype = _f64
    L.otf_model_completion_time.argtypes = [_P(_f64), _P(_f64), _i32, _f64, _f64, _f64, _f64, _i64]
    L.otf_model_select_quality.restype = _i32
    L.otf_model_select_quality.argtypes = [_f64, _i32, _i32, _f64, _P(_i64), _i32, _f64, _f64, _f64]
    L.otf_model_buffer_run.restype = ctypes.c_int
    L.otf_model_buffer_run.argtypes = [_f64, _i32, _P(_i32), _P(_f64), _P(_f64), _f64, _f64, _P(_f64)]
    L.otf_model_exact_sum.restype = ctypes.c_int
    L.otf_model_exact_sum.argtypes = [_P(_f64), _i64, _P(_f64)]
    L.otf_model_completion_times.restype = ctypes.c_int
    L.otf_model_completion_times.argtypes = [_vp, _vp, _i32, _f64, _f64, _f64, _vp, _vp, _i32, _vp, _vp]
    L.otf_gen_sizes.restype = ctypes.c_int
    L.otf_gen_sizes.argtypes = [_vp, _i32, _i64, _vp, _vp, _vp, _vp]
    L.otf_gen_tables.restype = ctypes.c_int
    L.otf_gen_tables.argtypes = [_vp, _i32, _i64, _vp, _vp]
    L.otf_model_libm.restype = ctypes.c_int
    L.otf_model_libm.argtypes = [_i32, _vp, _i64, _vp]
    L.otf_model_libm_dev.restype = ctypes.c_int
    L.otf_model_libm_dev.argtypes = [_i32, _vp, _i64, _vp, _vp]
    L.otf_run_batch.restype = ctypes.c_int
    L.otf_run_batch.argtypes = [_P(Batch), _i32, _vp]
    L.otf_run_summary.restype = ctypes.c_int
    L.otf_run_summary.argtypes = [_P(Batch), _i32, _vp]
    if L.otf_version() != ABI_VERSION:
        raise OtfError(f"libotfgpu ABI {L.otf_version()} != {ABI_VERSION}")
    for name, st in (("otf_sizeof_scenario", Scenario), ("otf_sizeof_batch", Batch), ("otf_sizeof_qoe", Qoe)):
        if getattr(L, name)() != ctypes.sizeof(st):
            raise OtfError(f"{name}: C {getattr(L, name)()} != ctypes {ctypes.sizeof(st)}")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().otf_last_error().decode("utf-8", "replace")
        raise (ValueError if rc == 1 else OtfError)(f"{what} failed ({rc}): {msg}")
