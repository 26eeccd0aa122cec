// otf_engine_common.cuh -- scenario view + client-side logic shared by engines.
//
// `Scn` binds one otf_scenario to its tables and output slices.  The client_*
// helpers are the parts of run_session (client.py:229-305) and client_proc
// (orchestrator.py:336-348) that only touch the client's own state, so the
// exact engine and the windowed engine run literally the same code for them.
#pragma once
#include <math.h>
#include <stdint.h>

#include "otf_model.cuh"
#include "otf_rng.cuh"
#include "otf_state.cuh"
#include "otfgpu.h"

namespace otf {

struct EngineState {                 // first 256 B of every scenario arena
    int64_t req_counter;             // MediaServer._ids (server.py:56)
    int64_t n_req, n_sess, n_seg, n_job;
    int64_t cur_bytes, entries;      // SegmentCache.current_bytes / len()
    int32_t lru_head, lru_tail;      // OrderedDict ends: head = oldest
    int32_t status;
    int32_t pad;
};

__device__ __forceinline__ void qoe_zero(QoeAcc *a, int lane, int nlanes) {
    uint32_t *p = (uint32_t *)a;
    for (int i = lane; i < (int)(sizeof(QoeAcc) / 4); i += nlanes) p[i] = 0;
}

struct Scn {
    const otf_batch *b;              // shared memory (windowed) or a local copy (exact)
    const otf_scenario *sc;          // shared memory (windowed) or global (exact)
    int32_t s;
    EngineState *st;
    int64_t *stats;
    otf_qoe *q;                      // final destination (global)
    QoeAcc *qa;                      // counters while running (shared or scratch)
    ClientCold *cold;                         // [n_clients] pick streams + registration times (scratch)
    double *tail_lat;                         // summary tails (otf_batch.tail_*)
    otf_sess_ent *tail_sess;
    double *tail_sup;
    uint64_t mag_g, mag_rg;                   // d / max_nseg, d / (n_ranks * max_nseg) by multiply-high
    double inv_grid_step;                     // 1 / sc->grid_step (0 when the trace grid is irregular)
    // the client model's constants in registers (read on every event; a shared-memory
    // reload after each atomic would sit on the client's dependency chain)
    double panic, safe, headroom, alpha, startup, resume;
    uint32_t div_g, div_rg;
    const int64_t *sizes, *bitrates, *manifest_b;
    const int32_t *segcounts;
    const double *seqdur, *segdur, *rho, *zipf, *starts, *values, *pbits, *arrivals, *eps;
    bool records;

    __device__ void init(const otf_batch *bb, const otf_scenario *scp, int32_t si) {
        b = bb;
        s = si;
        sc = scp;
        st = (EngineState *)(b->scratch + sc->scratch_off);
        stats = b->stats + (int64_t)si * OTF_ST_NSLOTS;
        q = b->qoe + si;
        sizes = b->i64_pool + sc->off_sizes;
        bitrates = b->i64_pool + sc->off_bitrates;
        manifest_b = b->i64_pool + sc->off_manifest;
        segcounts = b->i32_pool + sc->off_segcount;
        seqdur = b->f64_pool + sc->off_seqdur;
        segdur = b->f64_pool + sc->off_segdur;
        rho = b->f64_pool + sc->off_rho;
        zipf = b->f64_pool + sc->off_zipf;
        starts = b->f64_pool + sc->off_starts;
        values = b->f64_pool + sc->off_values;
        pbits = b->f64_pool + sc->off_pbits;
        arrivals = b->f64_pool + sc->off_arrivals;
        eps = b->f64_pool + sc->off_eps;
        tail_lat = b->tail_lat ? b->tail_lat + sc->lat_off : nullptr;
        tail_sess = b->tail_sess ? b->tail_sess + sc->ses_off : nullptr;
        tail_sup = b->tail_sup ? b->tail_sup + sc->sup_off : nullptr;
        records = b->mode == OTF_MODE_RECORDS;
        div_g = (uint32_t)sc->max_nseg;
        div_rg = (uint32_t)(sc->n_ranks * sc->max_nseg);
        mag_g = 0xffffffffffffffffull / div_g + 1ull;
        mag_rg = 0xffffffffffffffffull / div_rg + 1ull;
        inv_grid_step = sc->grid_step > 0 ? 1.0 / sc->grid_step : 0.0;
        panic = sc->panic; safe = sc->safe; headroom = sc->headroom;
        alpha = sc->alpha; startup = sc->startup; resume = sc->resume;
    }
    // floor(d / div) = umul64hi(d, floor((2^64-1)/div) + 1), exact for d, div < 2^31
    __device__ __forceinline__ uint32_t qdiv(uint32_t d, uint64_t mag, uint32_t) const {
        return (uint32_t)__umul64hi((uint64_t)d, mag);
    }

    // zero the scenario's outputs and counters (call once, single thread)
    __device__ void reset_outputs() {
        EngineState z = {};
        z.lru_head = z.lru_tail = -1;
        *st = z;
        for (int i = 0; i < OTF_ST_NSLOTS; i++) stats[i] = 0;
        qoe_zero(qa, 0, 1);
    }

    // write the final otf_qoe; the summary pass (otf_summary.cu) adds the
    // latency sum, the order statistics and the registration-order stall sum
    __device__ void flush_qoe() const {
        int64_t n_req = 0;
        for (int i = 0; i < OTF_LAT_BINS; i++) q->lat_hist[i] = qa->lat_hist[i];
        for (int i = 0; i < 8; i++) { q->path_count[i] = qa->path_count[i]; n_req += qa->path_count[i]; }
        for (int i = 0; i < OTF_STALL_BINS; i++) q->stall_hist[i] = 0;
        for (int i = 0; i < OTF_RANK_BINS; i++) q->rank_count[i] = qa->rank_count[i];
        q->n_requests = n_req; q->n_sessions = qa->n_ses_tail; q->n_segments = qa->n_segments;
        q->n_finished = 0; q->n_started = qa->n_sup_tail; q->n_stalls = 0;
        q->latency_sum = 0.0; q->stall_time_sum = 0.0; q->startup_delay_sum = 0.0;
        q->latency_p50 = 0.0; q->latency_p99 = 0.0;
        q->n_lat_tail = qa->n_lat_tail; q->n_stall_tail = 0;
        q->summary_flags = qa->flags;
    }

    // a nonzero request latency: kept for the order statistics and the exact sum
    __device__ __forceinline__ void tail_latency(double lat) {
        const uint32_t pos = atomicAdd(&qa->n_lat_tail, 1u);
        if (pos < (uint64_t)sc->lat_cap) tail_lat[pos] = lat;
        else flag(OTF_S_TAIL_OVERFLOW);
    }
    // playback started: the startup delay (client.py:128-131) is final
    __device__ __forceinline__ void tail_startup(double startup) {
        const uint32_t pos = atomicAdd(&qa->n_sup_tail, 1u);
        if (pos < (uint64_t)sc->sup_cap) tail_sup[pos] = startup;
        else flag(OTF_S_TAIL_OVERFLOW);
    }
    // a session's numbers are final (finished, aborted or harvested): its record
    __device__ __forceinline__ void tail_session(double reg_time, double stall_time, int32_t sid, uint32_t stalls,
                                                 bool finished) {
        const uint32_t pos = atomicAdd(&qa->n_ses_tail, 1u);
        if (pos < (uint64_t)sc->ses_cap) {
            otf_sess_ent e;
            e.reg_time = reg_time;
            e.stall_time = stall_time;
            e.sid = sid;
            e.stalls = stalls | (finished ? OTF_SE_FINISHED : 0u);
            tail_sess[pos] = e;
        } else {
            flag(OTF_S_TAIL_OVERFLOW);
        }
    }

    __device__ __forceinline__ int64_t &stat(int i) { return stats[i]; }
    __device__ __forceinline__ void flag(int32_t bits) { atomicOr(&st->status, bits); }
    __device__ __forceinline__ int32_t desc_id(int32_t seq, int32_t rank, int32_t index) const {
        return (seq * sc->n_ranks + (rank - 1)) * sc->max_nseg + index;
    }
    __device__ __forceinline__ int64_t size(int32_t d) const { return sizes[d]; }
    __device__ __forceinline__ int32_t segcount(int32_t seq) const { return segcounts[seq]; }
    __device__ __forceinline__ bool stored(int32_t rank) const { return (sc->stored_mask >> rank) & 1u; }
    __device__ __forceinline__ double arrival(int32_t cid) const { return arrivals[cid]; }
    __device__ __forceinline__ int64_t manifest(int32_t seq) const { return manifest_b[seq]; }
    __device__ __forceinline__ Trace trace(int32_t cid) const {
        Trace t;
        if (sc->off_tr_i >= 0) {                       // CSV traces: each client's own table
            const int64_t *ti = b->i64_pool + sc->off_tr_i + 3 * (int64_t)cid;
            const double *tf = b->f64_pool + sc->off_tr_f + 3 * (int64_t)cid;
            t.starts = b->f64_pool + ti[0];
            t.values = b->f64_pool + ti[1];
            t.n = (int32_t)ti[2];
            t.period = tf[0];
            t.pbits = tf[1];
            t.grid = tf[2];
            t.inv_grid = t.grid > 0 ? 1.0 / t.grid : 0.0;
            return t;
        }
        t.starts = starts;
        t.values = values + (int64_t)cid * sc->n_samples;
        t.period = sc->period;
        t.grid = sc->grid_step;
        t.inv_grid = inv_grid_step;
        t.pbits = pbits[cid];
        t.n = sc->n_samples;
        return t;
    }
    __device__ __forceinline__ int32_t desc_seq(int32_t d) const { return (int32_t)qdiv(d, mag_rg, div_rg); }
    __device__ __forceinline__ int32_t desc_rank(int32_t d) const {
        return (int32_t)(qdiv(d, mag_g, div_g) - (uint32_t)desc_seq(d) * (uint32_t)sc->n_ranks) + 1;
    }
    __device__ __forceinline__ int32_t desc_index(int32_t d) const {
        return (int32_t)((uint32_t)d - qdiv(d, mag_g, div_g) * div_g);
    }

    // Backend._enqueue bookkeeping: TranscodeJob + jobs.append (backend.py:156-170)
    __device__ int32_t record_job(int32_t d, int32_t origin, double now) {
        int64_t j = st->n_job++;
        stats[OTF_ST_JOBS_TOTAL]++;
        stats[origin == OTF_ORIGIN_DEMAND ? OTF_ST_JOBS_DEMAND : OTF_ST_JOBS_SPEC]++;
        if (records) {
            if (j < sc->job_cap) {
                int64_t o = sc->job_off + j;
                b->job_seq[o] = desc_seq(d);
                b->job_rep[o] = desc_rank(d);
                b->job_index[o] = desc_index(d);
                b->job_origin[o] = origin;
                b->job_outcome[o] = OTF_OUTCOME_PENDING;
                b->job_enq[o] = now;
                b->job_start[o] = NAN;
                b->job_fin[o] = NAN;
            } else {
                flag(OTF_S_RECORD_OVERFLOW);
            }
        }
        return (int32_t)j;
    }
    __device__ __forceinline__ void job_outcome(int32_t j, int32_t o) {
        if (records && j < sc->job_cap) b->job_outcome[sc->job_off + j] = o;
    }
    __device__ __forceinline__ void job_started(int32_t j, double now) {
        if (records && j < sc->job_cap) b->job_start[sc->job_off + j] = now;
    }
    __device__ __forceinline__ void job_finished(int32_t j, double now) {
        if (records && j < sc->job_cap) {
            b->job_fin[sc->job_off + j] = now;
            b->job_outcome[sc->job_off + j] = OTF_OUTCOME_COMPLETED;
        }
    }

    // ServiceSampler.service_time (transcode.py:95-99): the worker's own noise stream
    __device__ double service_time(Worker &k, int32_t wid, int32_t d) {
        int32_t rank = desc_rank(d), seq = desc_seq(d), idx = desc_index(d);
        double duration = seg_duration(seqdur[seq], segdur[seq], idx);
        double e = 0.0;
        if (sc->noise > 0) {
            if (k.eps_pos >= sc->eps_stride) flag(OTF_S_EPS_OVERFLOW);
            else e = eps[(int64_t)wid * sc->eps_stride + k.eps_pos];
            k.eps_pos++;
        }
        double svc = rho[rank - 1] * duration * (1.0 + e);
        return (1e-9 > svc) ? 1e-9 : svc;
    }

    // MediaServer.segment record append (server.py:76-77) + QoE epilogue
    __device__ void record_request(const Client &c, double response) {
        int64_t r = st->n_req++;
        if (records) {
            if (r < sc->req_cap) {
                int64_t o = sc->req_off + r;
                b->req_id[o] = c.req_id;
                b->req_seq[o] = c.seq;
                b->req_rep[o] = c.rank;
                b->req_index[o] = c.index;
                b->req_path[o] = c.path;
                b->req_arrival[o] = c.arrival;
                b->req_response[o] = response;
                b->req_bytes[o] = c.size;
            } else {
                flag(OTF_S_RECORD_OVERFLOW);
            }
        }
        double lat = response - c.arrival;
        qa->lat_hist[lat_bin(lat)]++;
        qa->path_count[c.path]++;
        if (lat != 0.0) tail_latency(lat);
    }

    __device__ void sync_session(const Client &c, double now) {      // _sync_report (client.py:284-288)
        if (!records || c.session >= sc->sess_cap) return;
        int64_t o = sc->sess_off + c.session;
        b->sess_end[o] = now;
        b->sess_stalls[o] = c.buf.stall_events;
        b->sess_stall_time[o] = c.buf.stall_time;
        b->sess_startup[o] = isnan(c.buf.started_at) ? NAN : c.buf.started_at - c.buf.session_start;
    }

    // session QoE, once per session when its numbers are final (the report as
    // _sync_report left it, client.py:284-288); the work is out of line with
    // scalar arguments (session closes are rare next to client events)
    __device__ __forceinline__ void qoe_session(const Client &c, int32_t cid, bool finished) {
        if (c.buf_live && !isnan(c.buf.started_at)) tail_startup(c.buf.started_at - c.buf.session_start);
        tail_session(cold[cid].reg_time, c.buf_live ? c.buf.stall_time : 0.0, c.session,
                     c.buf_live ? (uint32_t)c.buf.stall_events : 0u, finished);
    }

    __device__ void finish() {
        stats[OTF_ST_CACHE_CAPACITY] = sc->cache_capacity;
        stats[OTF_ST_CURRENT_BYTES] = st->cur_bytes;
        stats[OTF_ST_ENTRIES] = st->entries;
        stats[OTF_ST_STATUS] = st->status;
        int64_t *cnt = b->counts + (int64_t)s * 4;
        cnt[0] = st->n_req; cnt[1] = st->n_sess; cnt[2] = st->n_seg; cnt[3] = st->n_job;
        b->status[s] = st->status;
    }
};

// ---- client-local pieces -------------------------------------------------------

__device__ __forceinline__ void client_init(Client &c) {
    Client z = {};
    z.pc = C_START;
    z.session = -1;
    z.wait_next = -1;
    z.buf.started_at = NAN;
    c = z;
}

// orchestrator.py:338-340: the client's own pick stream
// Session-start RNG work runs once per session: kept out of line (plain
// pointer/scalar arguments, so nothing is forced onto the stack).
static __device__ __noinline__ void seed_picks(Pcg64 *g, uint64_t seed, int32_t cid) {
    uint32_t ent[8];
    int m = 0;
    m = push_words(ent, m, seed);
    m = push_words(ent, m, 3u);
    m = push_words(ent, m, (uint64_t)cid);
    pcg_seed(*g, ent, m);
}

// orchestrator.py:342 picks.integers(n); Zipf extension: inverse CDF on picks.random()
static __device__ __noinline__ int32_t draw_sequence(Pcg64 *g, int32_t n_seq, int32_t popularity, const double *zipf) {
    if (popularity == OTF_POP_ZIPF) {
        double u = pcg_next_double(*g);
        int32_t lo = 0, hi = n_seq - 1;                // first k with u < cdf[k] (else the last)
        while (lo < hi) {
            int32_t mid = (lo + hi) >> 1;
            if (u < zipf[mid]) hi = mid; else lo = mid + 1;
        }
        return lo;
    }
    return pcg_integers(*g, (uint32_t)n_seq);
}

__device__ __forceinline__ void client_arrive(Scn &S, Client &c, int32_t cid) {
    seed_picks(&S.cold[cid].picks, S.sc->seed, cid);
}

// orchestrator.py:341-345 + client.py:237-239: pick a sequence, register a report
__device__ inline void client_new_session(Scn &S, Client &c, int32_t cid, double now) {
    int32_t seq = draw_sequence(&S.cold[cid].picks, S.sc->n_seq, S.sc->popularity, S.zipf);
    S.cold[cid].reg_time = now;                        // registration order (client.py:237-239)
    c.seq = seq;
    int64_t sid = atomicAdd((unsigned long long *)&S.st->n_sess, 1ull);
    c.session = (int32_t)sid;
    c.buf_live = 0;
    c.sess_open = 1;
    if (S.records) {
        if (sid < S.sc->sess_cap) {
            int64_t o = S.sc->sess_off + sid;
            S.b->sess_client[o] = cid;
            S.b->sess_seq[o] = seq;
            S.b->sess_start[o] = now;
            S.b->sess_end[o] = 0.0;
            S.b->sess_stalls[o] = 0;
            S.b->sess_stall_time[o] = 0.0;
            S.b->sess_startup[o] = NAN;
            S.b->sess_flags[o] = 0;
        } else {
            S.flag(OTF_S_RECORD_OVERFLOW);
        }
    }
}

// client.py:245-248
__device__ __forceinline__ void client_start_playback(Client &c, double now) {
    buf_reset(c.buf, now);
    c.buf_live = 1;
    c.has_est = 0;
    c.est = 0.0;
    c.rank = 1;
    c.index = 0;
}

// client.py:255-256
__device__ __forceinline__ void client_select(Scn &S, Client &c) {
    if (c.index > 0)
        c.rank = select_quality(c.buf.level, c.rank, c.has_est != 0, c.est, S.bitrates, S.sc->n_ranks,
                                S.panic, S.safe, S.headroom);
}

// client.py:261-268; returns true when the session has more segments, else
// leaves the buffer advanced for the final sleep(level) (client.py:270-271).
__device__ inline bool client_segment_done(Scn &S, Client &c, double now) {
    double dt = now - c.xfer_start;                       // SegmentFetch.rate_bps
    double rate = dt > 0 ? ((double)c.size * 8.0) / dt : INFINITY;
    if (!c.has_est) { c.est = rate; c.has_est = 1; }
    else c.est = S.alpha * rate + (1.0 - S.alpha) * c.est;
    double duration = seg_duration(S.seqdur[c.seq], S.segdur[c.seq], c.index);
    buf_on_segment(c.buf, now, duration, S.startup, S.resume);
    int64_t g = atomicAdd((unsigned long long *)&S.st->n_seg, 1ull);
    if (S.records) {
        if (g < S.sc->seg_cap) {
            int64_t o = S.sc->seg_off + g;
            S.b->seg_session[o] = c.session;
            S.b->seg_index[o] = c.index;
            S.b->seg_rep[o] = c.rank;
            S.b->seg_start[o] = c.requested;
            S.b->seg_end[o] = now;
        } else {
            S.flag(OTF_S_RECORD_OVERFLOW);
        }
    }
    if (c.rank >= OTF_RANK_BINS) atomicOr(&S.qa->flags, (uint32_t)OTF_Q_RANKS_CAPPED);
    atomicAdd(&S.qa->rank_count[c.rank < OTF_RANK_BINS ? c.rank : OTF_RANK_BINS - 1], 1u);
    atomicAdd(&S.qa->n_segments, 1u);
    S.sync_session(c, now);
    c.index++;
    if (c.index < S.segcount(c.seq)) return true;
    buf_advance(c.buf, now);
    return false;
}

// client.py:272-280 (+ the finally clause)
__device__ inline void client_finish_session(Scn &S, Client &c, int32_t cid, double now) {
    buf_advance(c.buf, now);
    c.buf.phase = PH_FINISHED;
    if (S.records && c.session < S.sc->sess_cap) S.b->sess_flags[S.sc->sess_off + c.session] |= 1;
    S.sync_session(c, now);
    S.qoe_session(c, cid, true);
    c.buf_live = 0;
    c.sess_open = 0;
}

// Session given up after the last retry (client.py:257-260 + the finally
// clause): flagged aborted, synced without advancing the buffer.
__device__ inline void client_abort_session(Scn &S, Client &c, int32_t cid, double now) {
    if (S.records && c.session < S.sc->sess_cap) S.b->sess_flags[S.sc->sess_off + c.session] |= 2;
    S.sync_session(c, now);
    S.qoe_session(c, cid, false);
    c.buf_live = 0;
    c.sess_open = 0;
}

// SessionReport.harvest at the horizon (orchestrator.py:357-359, client.py:177-187)
__device__ inline void client_harvest(Scn &S, Client &c, int32_t cid, double horizon) {
    if (c.pc == C_HUNG) S.flag(OTF_S_HUNG);
    if (!c.sess_open) return;
    if (c.buf_live) {
        buf_advance(c.buf, horizon);
        S.sync_session(c, horizon);
    }
    S.qoe_session(c, cid, false);
}

}  // namespace otf
