"""Device driver: uploads a lowered batch, runs the engines, collects results.

This is the body behind the drop-in ``run_experiment`` (orchestrator.py:327-370)
and the batched sweep entry ``run_batch``.  Torch is used only to own device
memory and streams; all compute is libotfgpu.so (csrc/).  There is no CPU
path: without a CUDA device or without the library these functions raise.
"""

from __future__ import annotations

import ctypes
import dataclasses
import logging

import numpy as np
import torch

from . import _lib
from .inputs import BatchInputs, build_inputs
from .results import ExperimentResult

__all__ = ["DeviceBatch", "BatchResult", "run_batch", "run_experiment", "require_cuda"]

_log = logging.getLogger(__name__)
_NP = {"i8": np.int64, "i4": np.int32, "f8": np.float64}
_TORCH = {"i8": torch.int64, "i4": torch.int32, "f8": torch.float64}
_REC_GROUP = {"req": 0, "sess": 1, "seg": 2, "job": 3}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.OtfError("no CUDA device: the otfgpu engine has no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise _lib.OtfError(f"otfgpu runs on CUDA devices only, got {dev}")
    return dev


def _u8(ct) -> torch.Tensor:
    return torch.frombuffer(bytearray(bytes(ct)), dtype=torch.uint8)


class DeviceBatch:
    """One lowered batch resident in HBM, ready to launch (repeatedly)."""

    def __init__(self, inp: BatchInputs, device=None, pin: bool = False):
        self.inp = inp
        self.device = require_cuda(device)
        self.lib = _lib.lib()
        n = len(inp.lowered)
        self.n = n
        dev = self.device
        self.h_scen = _u8(inp.scenarios)
        self.h_tables = _u8(inp.size_tables)
        self.h_gen = _u8(inp.gen_jobs) if inp.gen_jobs is not None else torch.zeros(1, dtype=torch.uint8)
        self.h_f64 = torch.from_numpy(inp.f64)
        self.h_i64 = torch.from_numpy(inp.i64)
        self.h_i32 = torch.from_numpy(inp.i32)
        if pin:
            self.h_scen, self.h_tables, self.h_gen = (self.h_scen.pin_memory(), self.h_tables.pin_memory(),
                                                      self.h_gen.pin_memory())
            if not inp.pinned:
                self.h_f64, self.h_i64, self.h_i32 = (self.h_f64.pin_memory(), self.h_i64.pin_memory(),
                                                      self.h_i32.pin_memory())
        self.scen = torch.empty_like(self.h_scen, device=dev)
        self.tables = torch.empty_like(self.h_tables, device=dev)
        self.gen = torch.empty_like(self.h_gen, device=dev)
        # f64 pool = [device-generated prefix | host part]
        self.f64 = torch.empty(inp.f64_dev + self.h_f64.numel(), dtype=torch.float64, device=dev)
        self.f64_host = self.f64[inp.f64_dev:]
        self.i64 = torch.empty_like(self.h_i64, device=dev)
        self.i32 = torch.empty_like(self.h_i32, device=dev)
        self.scratch = torch.empty(inp.scratch_bytes, dtype=torch.uint8, device=dev)
        self.rec = {}
        if inp.mode == _lib.MODE_RECORDS:
            for name, dt in _lib.RECORD_FIELDS:
                total = inp.rec_totals[_REC_GROUP[name.split("_")[0]]]
                self.rec[name] = torch.empty(max(1, total), dtype=_TORCH[dt], device=dev)
        # summary tails (device only; the summary pass reduces them into the QoE blocks)
        self.tail_lat = torch.empty(max(1, inp.tail_totals[0]), dtype=torch.float64, device=dev)
        self.tail_sess = torch.empty(max(1, inp.tail_totals[1]) * _lib.SESS_ENT_BYTES, dtype=torch.uint8, device=dev)
        self.tail_sup = torch.empty(max(1, inp.tail_totals[2]), dtype=torch.float64, device=dev)
        self.counts = torch.zeros((n, 4), dtype=torch.int64, device=dev)
        self.stats = torch.zeros((n, _lib.ST_NSLOTS), dtype=torch.int64, device=dev)
        self.qoe = torch.zeros((n, ctypes.sizeof(_lib.Qoe) // 8), dtype=torch.int64, device=dev)
        self.status = torch.zeros(n, dtype=torch.int32, device=dev)
        b = _lib.Batch()
        b.n_scenarios, b.mode = n, inp.mode
        b.scenarios, b.f64_pool, b.i64_pool, b.i32_pool = (self.scen.data_ptr(), self.f64.data_ptr(),
                                                           self.i64.data_ptr(), self.i32.data_ptr())
        b.scratch = self.scratch.data_ptr()
        for name, _ in _lib.RECORD_FIELDS:
            setattr(b, name, self.rec[name].data_ptr() if name in self.rec else None)
        b.counts, b.stats = self.counts.data_ptr(), self.stats.data_ptr()
        b.qoe, b.status = self.qoe.data_ptr(), self.status.data_ptr()
        b.tail_lat, b.tail_sess, b.tail_sup = (self.tail_lat.data_ptr(), self.tail_sess.data_ptr(),
                                               self.tail_sup.data_ptr())
        # launch groups: scenarios of similar shared-memory size together (a big
        # scenario must not shrink everyone's occupancy), longest first within a group
        cost = np.array([l.cfg.clients * l.cfg.horizon_s / min(l.seq_segdur) for l in inp.lowered])
        smem = np.array(inp.smem_per if inp.smem_per else [inp.shared_bytes] * n, dtype=np.int64)
        cls = np.ceil(np.maximum(smem, 1) / 8192.0).astype(np.int64)
        order = np.lexsort((-cost, cls)).astype(np.int32)   # by class, then longest first
        self.order = torch.from_numpy(order).to(dev)
        self.groups = []
        # the group holding the longest scenario launches first: its CTAs reach the SMs
        # first, and the groups' kernels then run concurrently around it -- unless its
        # scenarios are >= 2x longer than every other group's: then it runs alone and the
        # rest follow it (co-located kernels slow its critical path by more than the
        # rest takes: config 4's 10,000-client class, 1.5 s alone vs 2.5 s co-located)
        classes = sorted(np.unique(cls), key=lambda c: -cost[cls == c].max())
        gmax = [float(cost[cls == c].max()) for c in classes]
        self.lead_alone = len(classes) > 1 and gmax[0] >= 2.0 * gmax[1]
        for c in classes:
            idx = np.nonzero(cls[order] == c)[0]
            gb = _lib.Batch.from_buffer_copy(b)
            gb.n_scenarios = int(len(idx))
            gb.order = self.order.data_ptr() + 4 * int(idx[0])
            gb.shared_bytes = int(smem[order[idx]].max())
            gb.engine_flags = 0
            gb.concurrent = n                          # the groups run concurrently (side streams)
            self.groups.append(gb)
        b.order = self.order.data_ptr()
        b.shared_bytes = inp.shared_bytes
        b.concurrent = n
        self.batch = b
        self.streams = [torch.cuda.Stream(dev) for _ in self.groups[1:]]
        self.n_tables = sum(1 for t in inp.size_tables if t.n_seq > 0)
        self.n_gen = inp.gen_streams and len(inp.gen_jobs) or 0
        self.upload()

    @property
    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.h_scen, self.h_tables, self.h_gen, self.h_f64,
                                                           self.h_i64, self.h_i32))

    def upload(self, stream: torch.cuda.Stream | None = None) -> None:
        """Host -> device copy of every input table (non_blocking when pinned)."""
        with torch.cuda.stream(stream) if stream is not None else torch.cuda.device(self.device):
            for d, h in ((self.scen, self.h_scen), (self.tables, self.h_tables), (self.gen, self.h_gen),
                         (self.f64_host, self.h_f64), (self.i64, self.h_i64), (self.i32, self.h_i32)):
                d.copy_(h, non_blocking=h.is_pinned())

    def generate(self, stream: torch.cuda.Stream | None = None) -> None:
        """Enqueue request generation: the seeded trace / arrival / noise streams
        (otf_gen_tables) and the segment-size tables (otf_gen_sizes)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.n_gen:
            rc = self.lib.otf_gen_tables(self.gen.data_ptr(), self.n_gen, self.inp.gen_streams, self.f64.data_ptr(),
                                         s.cuda_stream)
            _lib.check(rc, "otf_gen_tables")
        if self.n_tables:
            rc = self.lib.otf_gen_sizes(self.tables.data_ptr(), self.n_tables, 0, self.i64.data_ptr(),
                                        self.f64.data_ptr(), self.i32.data_ptr(), s.cuda_stream)
            _lib.check(rc, "otf_gen_sizes")

    def launch(self, stream: torch.cuda.Stream | None = None, sizes: bool = True, summary: bool = True) -> None:
        """Enqueue request generation (unless sizes=False: the tables from the last
        launch are reused) + the engine (+ the summary pass unless summary=False;
        then launch_summary runs it) on `stream` (default: current)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        flags = 0 if summary else _lib.BF_ENGINE_ONLY
        self.batch.engine_flags = flags
        for gb in self.groups:
            gb.engine_flags = flags
        if sizes:
            self.generate(s)
        if len(self.groups) <= 1 or self.inp.engine != _lib.ENGINE_WINDOWED:
            rc = self.lib.otf_run_batch(ctypes.byref(self.batch), self.inp.engine, s.cuda_stream)
            _lib.check(rc, "otf_run_batch")
            return
        # size classes run concurrently on side streams, joined back to `s`: the side
        # streams wait for what precedes the launches (generation), not for group 0
        ready = torch.cuda.Event()
        ready.record(s)
        rc = self.lib.otf_run_batch(ctypes.byref(self.groups[0]), self.inp.engine, s.cuda_stream)
        _lib.check(rc, "otf_run_batch")
        if self.lead_alone:                            # the rest starts when the leading group ends
            ready = torch.cuda.Event()
            ready.record(s)
        for gb, st in zip(self.groups[1:], self.streams):
            st.wait_event(ready)
            rc = self.lib.otf_run_batch(ctypes.byref(gb), self.inp.engine, st.cuda_stream)
            _lib.check(rc, "otf_run_batch")
        for st in self.streams:
            s.wait_stream(st)

    def launch_summary(self, stream: torch.cuda.Stream | None = None) -> None:
        """The summary pass alone, after launch(summary=False) on the same stream."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(self.lib.otf_run_summary(ctypes.byref(self.batch), self.inp.engine, s.cuda_stream),
                   "otf_run_summary")

    def fetch(self) -> "BatchResult":
        torch.cuda.synchronize(self.device)
        counts = self.counts.cpu().numpy()
        stats = self.stats.cpu().numpy()
        status = self.status.cpu().numpy()
        qoe = self.qoe.cpu().numpy()
        rec = {k: v.cpu().numpy() for k, v in self.rec.items()}
        sizes = self.i64.cpu().numpy()
        return BatchResult(self.inp, counts, stats, status, qoe, rec, sizes)


def order_sessions(a: dict) -> None:
    """Put windowed-engine sessions in registration order (client.py:237-239).

    The windowed engine registers sessions from parallel lanes, so their slots
    come out in arbitrary order; registration order is start time order (ties
    are re-run on the exact engine).  Segment rows are re-pointed at the new
    session slots; per-session segment order is already append order."""
    perm = np.argsort(a["sess_start"], kind="stable")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    for k in ("sess_client", "sess_seq", "sess_stalls", "sess_flags", "sess_start", "sess_end",
              "sess_stall_time", "sess_startup"):
        a[k] = a[k][perm]
    if len(a["seg_session"]):
        a["seg_session"] = inv[a["seg_session"]].astype(np.int32)
        seg_order = np.argsort(a["seg_session"], kind="stable")
        for k in ("seg_session", "seg_index", "seg_rep", "seg_start", "seg_end"):
            a[k] = a[k][seg_order]


QOE_FIELDS = ("n_requests", "n_sessions", "n_segments", "n_finished", "n_started", "n_stalls", "latency_sum",
              "stall_time_sum", "startup_delay_sum", "latency_p50", "latency_p99", "n_lat_tail", "n_stall_tail",
              "summary_flags")


def parse_qoe(row: np.ndarray) -> dict:
    """One otf_qoe row (int64 words) as a dict of Python numbers / lists."""
    q = _lib.Qoe.from_buffer_copy(np.ascontiguousarray(row).tobytes())
    out = {"lat_hist": list(q.lat_hist), "path_count": list(q.path_count)[:5], "stall_hist": list(q.stall_hist),
           "rank_count": list(q.rank_count)}
    for f in QOE_FIELDS:
        out[f] = getattr(q, f)
    return out


@dataclasses.dataclass
class BatchResult:
    inp: BatchInputs
    counts: np.ndarray
    stats: np.ndarray
    status: np.ndarray
    qoe: np.ndarray
    rec: dict
    i64_pool: np.ndarray

    def arrays(self, i: int) -> dict:
        out = {}
        for name, _ in _lib.RECORD_FIELDS:
            g = _REC_GROUP[name.split("_")[0]]
            off = int(self.inp.rec_offsets[i, g])
            n = int(min(self.counts[i, g], self.inp.caps[i, g]))
            out[name] = self.rec[name][off:off + n].copy()
        if self.inp.engine == _lib.ENGINE_WINDOWED:
            order_sessions(out)
        return out

    def session_tie(self, i: int) -> bool:
        """Windowed engine: two sessions registered at the identical instant (order unknown)."""
        if self.inp.engine != _lib.ENGINE_WINDOWED or not self.rec:
            return False
        g = _REC_GROUP["sess"]
        off = int(self.inp.rec_offsets[i, g])
        n = int(min(self.counts[i, g], self.inp.caps[i, g]))
        st = np.sort(self.rec["sess_start"][off:off + n])
        return bool(n > 1 and (st[1:] == st[:-1]).any())

    def sizes(self, i: int) -> np.ndarray:
        sc = self.inp.scenarios[i]
        n = sc.n_seq * sc.n_ranks * sc.max_nseg
        return self.i64_pool[sc.off_sizes:sc.off_sizes + n].reshape(sc.n_seq, sc.n_ranks, sc.max_nseg)

    def result(self, i: int) -> ExperimentResult:
        low = self.inp.lowered[i]
        return ExperimentResult(low.cfg, self.arrays(i) if self.rec else {}, self.stats[i], low.seq_ids,
                                sizes=self.sizes(i), seq_dur=low.seq_dur, seq_segdur=low.seq_segdur,
                                qoe=self.qoe[i], status=int(self.status[i]), counts=self.counts[i])

    @property
    def total_requests(self) -> int:
        return int(self.counts[:, 0].sum())


def run_batch(configs, mode: str = "records", engine: str = "windowed", device=None,
              max_retries: int = 4, _caps=None, _eps_scale: float = 1.0, _tail_caps=None) -> list[ExperimentResult]:
    """Run every config on the GPU; returns one ExperimentResult per config.

    Scenarios whose record buffers or noise tables were too small are re-run
    with exact sizes; scenarios the windowed engine flags with an ordering tie
    are re-run on the exact engine.
    """
    require_cuda(device)                               # no CPU path: fail before any host work
    m = _lib.MODE_RECORDS if mode == "records" else _lib.MODE_HISTOGRAM
    eng = _lib.ENGINE_WINDOWED if engine == "windowed" else _lib.ENGINE_EXACT
    from .inputs import lower_any
    configs = [lower_any(c) for c in configs]          # validated and lowered once per call
    if m == _lib.MODE_RECORDS and _caps is None and len(configs) > 1:
        # record buffers grow with the requests (~212 B per expected request): a big
        # sweep in records mode runs in chunks that fit half the free device memory
        from .inputs import _default_caps
        dev = require_cuda(device)
        budget = torch.cuda.mem_get_info(dev)[0] // 2
        need = []
        for c in configs:
            r, s_, g, j = _default_caps(c)
            need.append(48 * r + 48 * s_ + 28 * g + 44 * j)
        if sum(need) > budget:
            out, chunk, used = [], [], 0
            for c, b in zip(configs, need):
                if chunk and used + b > budget:
                    out += run_batch(chunk, mode, engine, device, max_retries)
                    chunk, used = [], 0
                chunk.append(c)
                used += b
            return out + run_batch(chunk, mode, engine, device, max_retries)
    results: list = [None] * len(configs)
    todo = list(range(len(configs)))
    caps = {i: tuple(c) for i, c in enumerate(_caps)} if _caps is not None else {}   # test hook
    tcaps = {i: tuple(c) for i, c in enumerate(_tail_caps)} if _tail_caps is not None else {}   # test hook
    eps_scale = {i: _eps_scale for i in todo} if _eps_scale != 1.0 else {}         # test hook
    lcaps: dict = {}                                   # server-event list capacities after an overflow
    engines = {i: eng for i in todo}
    if eng == _lib.ENGINE_WINDOWED:                    # outside the windowed engine's limits: exact, up front
        from .inputs import windowed_fits
        limit = torch.cuda.get_device_properties(require_cuda(device)).shared_memory_per_block_optin
        for i in todo:
            ok, why = windowed_fits(configs[i], limit)
            if not ok:
                engines[i] = _lib.ENGINE_EXACT
                _log.warning("scenario %d runs on the exact engine (outside the windowed engine's limits: %s)",
                             i, why)
    for _attempt in range(max_retries + 1):
        if not todo:
            break
        groups = {}
        for i in todo:
            groups.setdefault((engines[i], eps_scale.get(i, 1)), []).append(i)
        nxt = []
        for (e, es), idx in groups.items():
            cap_list = [caps[i] if i in caps else None for i in idx]
            use_caps = None
            if any(c is not None for c in cap_list):
                inp0 = build_inputs([configs[i] for i in idx], engine=e, mode=m, eps_scale=es)
                use_caps = [c if c is not None else tuple(inp0.caps[k]) for k, c in enumerate(cap_list)]
            tail = [tcaps.get(i) for i in idx]
            lc = [lcaps.get(i, 0) for i in idx]
            inp = build_inputs([configs[i] for i in idx], engine=e, mode=m, caps=use_caps, eps_scale=es, pin=True,
                               tail_caps=tail if any(t is not None for t in tail) else None,
                               list_caps=lc if any(lc) else None)
            db = DeviceBatch(inp, device, pin=True)
            db.launch()
            br = db.fetch()
            for k, i in enumerate(idx):
                st = int(br.status[k])
                if st & _lib.S_INTERNAL:
                    raise _lib.OtfError(f"scenario {i}: engine invariant violated (status {st:#x})")
                retry = False
                if st & _lib.S_UNFIT:
                    _log.warning("scenario %d: outside the windowed engine's limits at run time "
                                 "(status %#x); re-running it on the exact engine", i, st)
                if st & _lib.S_LIST_OVERFLOW:             # a burst of simultaneous requests: a 4x list
                    if not _grow_list_cap(configs[i], lcaps, i, device):
                        engines[i] = _lib.ENGINE_EXACT
                    retry = True
                if st & (_lib.S_TIE | _lib.S_UNFIT) or (m == _lib.MODE_RECORDS and br.session_tie(k)):
                    engines[i] = _lib.ENGINE_EXACT
                    retry = True
                if st & _lib.S_EPS_OVERFLOW:
                    eps_scale[i] = eps_scale.get(i, 1) * 4
                    retry = True
                if st & _lib.S_RECORD_OVERFLOW:
                    caps[i] = tuple(int(x) + 1 for x in br.counts[k])
                    retry = True
                if st & _lib.S_TAIL_OVERFLOW:             # exact counts (the stalled ones bounded by
                    q = _lib.Qoe.from_buffer_copy(br.qoe[k].tobytes())   # the sessions if not yet known)
                    n_ses = int(q.n_sessions)
                    n_stl = int(q.n_stall_tail) if q.n_stall_tail else n_ses
                    tcaps[i] = (int(q.n_lat_tail) + 1, n_ses + 1, n_stl + 1, int(q.n_started) + 1)
                    retry = True
                if retry:
                    nxt.append(i)
                else:
                    results[i] = br.result(k)
                    results[i].engine = "exact" if e == _lib.ENGINE_EXACT else "windowed"
                    results[i].attempts = _attempt + 1
                    results[i].list_cap = lcaps.get(i, 0)
                    results[i].eps_scale = es
        todo = nxt
    if todo:
        raise _lib.OtfError(f"scenarios {todo} did not converge after {max_retries} retries")
    return results


def _grow_list_cap(cfg, lcaps: dict, i: int, device) -> bool:
    """Quadruple scenario i's server-event list (a power of two, at most 16,384
    entries and the device's shared memory); False when it cannot grow."""
    from .inputs import lower_any
    L = _lib.lib()
    low = lower_any(cfg)
    cur = lcaps.get(i) or int(L.otf_list_cap(low.cfg.clients))
    new = cur * 4
    limit = torch.cuda.get_device_properties(require_cuda(device)).shared_memory_per_block_optin
    smem = int(L.otf_shared_bytes_cap(low.cfg.clients, len(low.seq_ids), low.n_ranks, max(low.counts), new))
    if new > 16384 or smem > limit:
        _log.warning("scenario %d: %d simultaneous requests exceed the windowed engine's list; exact engine", i, cur)
        return False
    lcaps[i] = new
    return True


def run_experiment(config) -> ExperimentResult:
    """Drop-in for otfstream.orchestrator.run_experiment (orchestrator.py:327-370)."""
    return run_batch([config], mode="records")[0]
