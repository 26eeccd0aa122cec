/*
 * otf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's virtual-clock experiment
 * (otfstream.orchestrator.run_experiment, /root/reference/pkg/src/otfstream/
 * orchestrator.py:327-370) used as the parity checker for the CUDA engine in
 * paper_2603_08417_b200/csrc.  It is deliberately a straight, sequential
 * restatement of the reference's event loop: a (when, tick) timer heap plus a
 * FIFO ready queue (sim.py:280-360) driving explicit state machines for the
 * client coroutines (client.py:229-305, orchestrator.py:336-348) and the
 * worker coroutines (backend.py:186-216).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or
 * the timed CPU baseline -- never as part of the product path.
 *
 * Pinned against the reference itself: the tests/golden fixtures were produced by
 * running the unmodified reference (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks this file against them bit-for-bit.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no FMA contraction so
 * every double op rounds exactly like CPython's).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "otf_oracle.h"

/* ------------------------------------------------------------------------ */
/* numpy SeedSequence + PCG64 (numpy 2.3.5, numpy/random/bit_generator.pyx   */
/* SeedSequence.mix_entropy/generate_state; numpy/random/src/pcg64).  Used   */
/* by the reference at content.py:165-167 (segment sizes) and                */
/* orchestrator.py:340-342 (sequence picks).                                 */
/* ------------------------------------------------------------------------ */

#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

typedef unsigned __int128 u128;

typedef struct {
    u128 state, inc;
    int has_uint32;
    uint32_t uinteger;
} pcg64_t;

/* numpy's _int_to_uint32_array: little-endian 32-bit words, 0 -> [0]. */
static int push_words(uint32_t *w, int n, uint64_t v) {
    if (v == 0) { w[n++] = 0; return n; }
    while (v) { w[n++] = (uint32_t)(v & 0xffffffffu); v >>= 32; }
    return n;
}

static void seed_pcg64(pcg64_t *g, const uint32_t *ent, int m) {
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
#define HASHMIX(v_, out_) do { uint32_t _v = (v_); _v ^= hc; hc *= SS_MULT_A; _v *= hc; _v ^= _v >> 16; (out_) = _v; } while (0)
#define MIX(x_, y_, out_) do { uint32_t _r = SS_MIX_L * (x_) - SS_MIX_R * (y_); _r ^= _r >> 16; (out_) = _r; } while (0)
    for (int i = 0; i < 4; i++) { HASHMIX(i < m ? ent[i] : 0u, pool[i]); }
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) { uint32_t h; HASHMIX(pool[s], h); MIX(pool[d], h, pool[d]); }
    for (int s = 4; s < m; s++)
        for (int d = 0; d < 4; d++) { uint32_t h; HASHMIX(ent[s], h); MIX(pool[d], h, pool[d]); }
#undef HASHMIX
#undef MIX
    uint32_t st[8];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb; hb *= SS_MULT_B; v *= hb; v ^= v >> 16;
        st[i] = v;
    }
    uint64_t v0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    uint64_t v1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
    uint64_t v2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
    uint64_t v3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
    u128 seed = ((u128)v0 << 64) | v1;
    u128 inc = ((u128)v2 << 64) | v3;
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    g->state = 0;
    g->inc = (inc << 1) | 1u;
    g->state = g->state * mult + g->inc;
    g->state += seed;
    g->state = g->state * mult + g->inc;
    g->has_uint32 = 0;
    g->uinteger = 0;
}

static uint64_t pcg_next64(pcg64_t *g) {
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    g->state = g->state * mult + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t pcg_next32(pcg64_t *g) {
    if (g->has_uint32) { g->has_uint32 = 0; return g->uinteger; }
    uint64_t n = pcg_next64(g);
    g->has_uint32 = 1;
    g->uinteger = (uint32_t)(n >> 32);
    return (uint32_t)n;
}

static double pcg_next_double(pcg64_t *g) {
    return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* Generator.integers(n) for 1 <= n <= 2^32 (bounded Lemire, 32-bit path). */
static int64_t pcg_integers(pcg64_t *g, int64_t n) {
    uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    if (rng == 0xffffffffu) return pcg_next32(g);
    uint32_t r1 = rng + 1;
    uint64_t m = (uint64_t)pcg_next32(g) * r1;
    uint32_t left = (uint32_t)m;
    if (left < r1) {
        uint32_t thr = (uint32_t)(-r1) % r1;
        while (left < thr) { m = (uint64_t)pcg_next32(g) * r1; left = (uint32_t)m; }
    }
    return (int64_t)(m >> 32);
}

/* ------------------------------------------------------------------------ */
/* Inputs: traces (netem.py:39-64,179-202), sizes (content.py:204-218).      */
/* ------------------------------------------------------------------------ */

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* CPython >= 3.12 builtin sum() over floats (Neumaier compensation). */
static double py_fsum_neumaier(const double *xs, int n) {
    double f = 0.0, c = 0.0;
    for (int i = 0; i < n; i++) {
        double x = xs[i];
        double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

int oracle_sample_times(double duration, double step, double *starts, int cap) {
    /* synthetic_trace: t = 0; while t < duration: ...; t += step (netem.py:195-201) */
    int n = 0;
    double t = 0.0;
    while (t < duration) {
        if (n < cap) starts[n] = t;
        n++;
        t += step;
    }
    return n;
}

/* One synthetic trace from its normal draws z[0..n] (netem.py:179-202) and its
 * BandwidthTrace period / period-bits (netem.py:39-64). */
static void build_trace(const oracle_scenario *sc, const double *z, const double *ts, int n,
                        double *values, double *period_out, double *pbits_out) {
    double x = sc->trace_mu + sc->trace_sigma * z[0];
    for (int i = 0; i < n; i++) {
        double e = exp(x);
        double bw = e > sc->trace_floor ? e : sc->trace_floor;   /* max(exp(x), floor) */
        bw = sc->trace_cap < bw ? sc->trace_cap : bw;           /* min(.., cap) */
        values[i] = bw;
        x = sc->trace_mu + (x - sc->trace_mu) * sc->trace_decay + sc->trace_spread * z[i + 1];
    }
    double tail = 1.0;
    if (n > 1) {
        double *g = (double *)malloc(sizeof(double) * (size_t)(n - 1));
        for (int i = 0; i + 1 < n; i++) g[i] = ts[i + 1] - ts[i];
        qsort(g, (size_t)(n - 1), sizeof(double), cmp_double);
        int m = n - 1;
        tail = (m & 1) ? g[m / 2] : (g[m / 2 - 1] + g[m / 2]) / 2.0;  /* statistics.median */
        free(g);
    }
    double period = ts[n - 1] + tail;
    double *terms = (double *)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; i++) {
        double end = (i + 1 < n) ? ts[i + 1] : period;
        terms[i] = values[i] * (end - ts[i]);
    }
    *pbits_out = py_fsum_neumaier(terms, n);
    *period_out = period;
    free(terms);
}

/* ------------------------------------------------------------------------ */
/* Event loop (sim.py:280-360).                                              */
/* ------------------------------------------------------------------------ */

typedef struct { double when; uint64_t tick; int32_t task; } timer_ent;

typedef struct { int32_t task; int64_t value; } ready_ent;

enum { PH_STARTUP = 0, PH_PLAYING = 1, PH_STALLED = 2, PH_FINISHED = 3 };

enum {
    C_START = 0, C_ARRIVED, C_SESSION, C_MAN_LAT, C_MAN_XFER, C_INDEX_HEAD, C_TARGET_WAIT,
    C_SEG_LAT, C_SEG_WAIT, C_SEG_XFER, C_PLAYOUT, C_DONE, C_HUNG, C_RETRY
};
enum { W_START = 0, W_NEXT, W_GOT, W_SERVICE, W_WOKEN };

typedef struct {
    int pc;
    int32_t seq, session, index, rank, has_est, buf_live;
    double est;
    /* PlayerBuffer (client.py:74-131) */
    double level, position, last_sync, stall_time, started_at, session_start;
    int32_t phase, stall_events;
    /* pending request */
    double requested, arrival, xfer_start;
    int64_t req_id, size;
    int32_t path, desc;
    int32_t attempt;                 /* _fetch_with_retry (client.py:291-305) */
    double backoff;
    int32_t wait_next;
    pcg64_t picks;
    const double *values, *starts;   /* the client's BandwidthTrace (netem.py:39-64) */
    double pbits, period;
    int32_t n_samples;
} client_t;

typedef struct { int pc; int32_t job; int64_t eps_pos; } worker_t;

typedef struct {
    const oracle_scenario *sc;
    oracle_outputs *out;
    double now;
    uint64_t tick;
    timer_ent *heap; int64_t heap_n;
    ready_ent *ready; int64_t rq_head, rq_n, rq_cap;
    client_t *cl; worker_t *wk;
    int32_t n_clients, n_workers, n_tasks;
    /* catalog */
    int64_t *sizes; int32_t *seg_count; int32_t n_desc;
    const double *starts; int32_t n_samples; double period;
    /* cache (cache.py:27-92) */
    int8_t *present; int32_t *lru_prev, *lru_next; int32_t lru_head, lru_tail;
    int64_t cur_bytes, entries;
    /* in-flight waiters (backend.py:125-133,209-216) */
    int8_t *inflight; int32_t *wq_head, *wq_tail;
    /* job FIFO + getter FIFO (sim.py:215-247) */
    int32_t *jq; int64_t jq_head, jq_n, jq_cap;
    int32_t *gq; int64_t gq_head, gq_n;
    /* demand-priority mode (backend.py:103-105,160-184): speculative FIFO + wakeup tokens */
    int32_t *sq; int64_t sq_head, sq_n;
    int64_t tokens;
    int64_t req_counter;
    const double *arrivals;
    int status;
} world_t;

static int tm_less(const timer_ent *a, const timer_ent *b) {
    return a->when < b->when || (a->when == b->when && a->tick < b->tick);
}

static void heap_push(world_t *w, double when, int32_t task) {
    int64_t i = w->heap_n++;
    timer_ent e = { when, w->tick++, task };
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!tm_less(&e, &w->heap[p])) break;
        w->heap[i] = w->heap[p];
        i = p;
    }
    w->heap[i] = e;
}

static timer_ent heap_pop(world_t *w) {
    timer_ent top = w->heap[0];
    timer_ent last = w->heap[--w->heap_n];
    int64_t i = 0, n = w->heap_n;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        const timer_ent *best = &last;
        if (l < n && tm_less(&w->heap[l], best)) { m = l; best = &w->heap[l]; }
        if (r < n && tm_less(&w->heap[r], best)) { m = r; best = &w->heap[r]; }
        if (m == i) break;
        w->heap[i] = w->heap[m];
        i = m;
    }
    if (n > 0) w->heap[i] = last;
    return top;
}

static void ready_push(world_t *w, int32_t task, int64_t value) {
    int64_t pos = (w->rq_head + w->rq_n) % w->rq_cap;
    w->ready[pos].task = task;
    w->ready[pos].value = value;
    w->rq_n++;
}

/* loop.sleep(delay) (sim.py:317-324): returns 1 when the caller must yield. */
static int do_sleep(world_t *w, int32_t task, double delay, int *pc_hung) {
    if (delay <= 0) return 0;
    if (isinf(delay)) { *pc_hung = 1; return 1; }
    heap_push(w, w->now + delay, task);
    return 1;
}

static inline int32_t desc_id(const world_t *w, int32_t seq, int32_t rank, int32_t index) {
    return (seq * w->sc->n_ranks + (rank - 1)) * w->sc->max_nseg + index;
}

static inline int is_stored(const world_t *w, int32_t rank) {
    return (w->sc->stored_mask >> rank) & 1u;
}

/* ---- cache (cache.py:45-81) ---- */
static void lru_unlink(world_t *w, int32_t d) {
    int32_t p = w->lru_prev[d], n = w->lru_next[d];
    if (p >= 0) w->lru_next[p] = n; else w->lru_head = n;
    if (n >= 0) w->lru_prev[n] = p; else w->lru_tail = p;
}
static void lru_append(world_t *w, int32_t d) {
    w->lru_prev[d] = w->lru_tail;
    w->lru_next[d] = -1;
    if (w->lru_tail >= 0) w->lru_next[w->lru_tail] = d; else w->lru_head = d;
    w->lru_tail = d;
}
static int cache_get(world_t *w, int32_t d) {
    if (!w->present[d]) { w->out->stats[ST_MISSES]++; return 0; }
    lru_unlink(w, d);
    lru_append(w, d);
    w->out->stats[ST_HITS]++;
    return 1;
}
static void cache_put(world_t *w, int32_t d) {
    int64_t size = w->sizes[d];
    int64_t cap = w->sc->cache_capacity;
    if (size > cap) { w->out->stats[ST_REJECTED]++; return; }
    if (w->present[d]) {
        w->cur_bytes -= w->sizes[d];
        lru_unlink(w, d);
        w->present[d] = 0;
        w->entries--;
    }
    while (w->cur_bytes + size > cap) {
        int32_t v = w->lru_head;
        lru_unlink(w, v);
        w->present[v] = 0;
        w->entries--;
        w->cur_bytes -= w->sizes[v];
        w->out->stats[ST_EVICTIONS]++;
    }
    lru_append(w, d);
    w->present[d] = 1;
    w->entries++;
    w->cur_bytes += size;
}

/* ---- backend (backend.py:135-216) ---- */
static void set_overflow(world_t *w) { w->status = ORACLE_EOVERFLOW; }

/* Backend._enqueue (backend.py:156-170): returns 1 on OverloadError (queue at
 * its bound and no idle worker: Queue.put_nowait raises QueueFull, sim.py:229-240). */
static int enqueue_job(world_t *w, int32_t d, int32_t origin) {
    oracle_outputs *o = w->out;
    const int prio = w->sc->demand_priority;
    if (prio) {
        /* workers never wait on the job queues in this mode, so a bounded demand queue
         * overflows on its own length (sim.py:238-239) */
        if (origin == ORIGIN_DEMAND && w->sc->queue_bound > 0 && w->jq_n >= w->sc->queue_bound) return 1;
    } else if (w->gq_n == 0 && w->sc->queue_bound > 0 && w->jq_n >= w->sc->queue_bound) {
        return 1;
    }
    int64_t j = o->n_job++;
    if (j < o->job_cap) {
        int32_t per_seq = w->sc->n_ranks * w->sc->max_nseg;
        o->job_seq[j] = d / per_seq;
        o->job_rep[j] = (d % per_seq) / w->sc->max_nseg + 1;
        o->job_index[j] = d % w->sc->max_nseg;
        o->job_origin[j] = origin;
        o->job_outcome[j] = OUT_PENDING;
        o->job_enq[j] = w->now;
        o->job_start[j] = NAN;
        o->job_fin[j] = NAN;
    } else {
        set_overflow(w);
    }
    o->stats[ST_JOBS_TOTAL]++;
    o->stats[origin == ORIGIN_DEMAND ? ST_JOBS_DEMAND : ST_JOBS_SPEC]++;
    w->inflight[d] = 1;
    w->wq_head[d] = -1;
    w->wq_tail[d] = -1;
    if (prio) {
        if (origin == ORIGIN_SPEC) {
            w->sq[(w->sq_head + w->sq_n) % w->jq_cap] = (int32_t)j;
            w->sq_n++;
        } else {
            w->jq[(w->jq_head + w->jq_n) % w->jq_cap] = (int32_t)j;
            w->jq_n++;
        }
        /* _wakeup.put_nowait(None, force=True): wake the first idle worker or leave a token */
        if (w->gq_n > 0) {
            int32_t wid = w->gq[w->gq_head];
            w->gq_head = (w->gq_head + 1) % w->n_workers;
            w->gq_n--;
            ready_push(w, wid, -1);
        } else {
            w->tokens++;
        }
        return 0;
    }
    /* Queue.put_nowait: hand to the first waiting getter, else append. */
    if (w->gq_n > 0) {
        int32_t wid = w->gq[w->gq_head];
        w->gq_head = (w->gq_head + 1) % w->n_workers;
        w->gq_n--;
        ready_push(w, wid, j);
    } else {
        if (w->jq_n >= w->jq_cap) { set_overflow(w); return 0; }
        w->jq[(w->jq_head + w->jq_n) % w->jq_cap] = (int32_t)j;
        w->jq_n++;
    }
    return 0;
}

static void maybe_speculate(world_t *w, int32_t seq, int32_t rank, int32_t index) {
    int64_t *st = w->out->stats;
    if (!w->sc->spec_enabled) { st[ST_SKIP_DISABLED]++; return; }
    int32_t ni = index + 1;
    if (ni >= w->seg_count[seq]) { st[ST_SKIP_EOS]++; return; }
    if (is_stored(w, rank)) { st[ST_SKIP_STORED]++; return; }
    int32_t d = desc_id(w, seq, rank, ni);
    if (w->sc->cache_enabled && w->present[d]) { st[ST_SKIP_CACHED]++; return; }
    if (w->inflight[d]) { st[ST_SKIP_INFLIGHT]++; return; }
    if (enqueue_job(w, d, ORIGIN_SPEC)) { st[ST_SKIP_OVERLOAD]++; return; }
    st[ST_SPEC_ENQUEUED]++;
}

static void resolve(world_t *w, int32_t d) {
    if (!w->inflight[d]) return;
    w->inflight[d] = 0;
    for (int32_t c = w->wq_head[d]; c >= 0; c = w->cl[c].wait_next)
        ready_push(w, w->n_workers + c, 0);
    w->wq_head[d] = w->wq_tail[d] = -1;
}

static void add_waiter(world_t *w, int32_t d, int32_t c) {
    w->cl[c].wait_next = -1;
    if (w->wq_tail[d] >= 0) w->cl[w->wq_tail[d]].wait_next = c; else w->wq_head[d] = c;
    w->wq_tail[d] = c;
}

/* ---- records ---- */
static void append_request(world_t *w, client_t *c, double response) {
    oracle_outputs *o = w->out;
    int64_t r = o->n_req++;
    if (r >= o->req_cap) { set_overflow(w); return; }
    int32_t per_seq = w->sc->n_ranks * w->sc->max_nseg;
    o->req_id[r] = c->req_id;
    o->req_seq[r] = c->desc / per_seq;
    o->req_rep[r] = c->rank;
    o->req_index[r] = c->index;
    o->req_path[r] = c->path;
    o->req_arrival[r] = c->arrival;
    o->req_response[r] = response;
    o->req_bytes[r] = c->size;
}

static void sync_report(world_t *w, client_t *c, double now) {
    oracle_outputs *o = w->out;
    int64_t s = c->session;
    if (s >= o->sess_cap) return;
    o->sess_end[s] = now;
    o->sess_stalls[s] = c->stall_events;
    o->sess_stall_time[s] = c->stall_time;
    o->sess_startup[s] = isnan(c->started_at) ? NAN : c->started_at - c->session_start;
}

/* PlayerBuffer.advance (client.py:91-112) */
static void buf_advance(client_t *c, double now) {
    double dt = now - c->last_sync;
    c->last_sync = now;
    if (c->phase == PH_PLAYING) {
        if (c->level >= dt - 1e-9) {
            double l = c->level - dt;
            c->level = (l > 0.0) ? l : 0.0;    /* max(0.0, level - dt) */
            c->position += dt;
        } else {
            double played = c->level;
            c->position += played;
            c->level = 0.0;
            c->phase = PH_STALLED;
            c->stall_events++;
            c->stall_time += dt - played;
        }
    } else if (c->phase == PH_STALLED) {
        c->stall_time += dt;
    }
}

/* PlayerBuffer.on_segment (client.py:114-121) */
static void buf_on_segment(const oracle_scenario *sc, client_t *c, double now, double duration) {
    buf_advance(c, now);
    c->level += duration;
    if (c->phase == PH_STARTUP && c->level >= sc->startup) {
        c->phase = PH_PLAYING;
        c->started_at = now;
    } else if (c->phase == PH_STALLED && c->level >= sc->resume) {
        c->phase = PH_PLAYING;
    }
}

/* select_quality (client.py:134-146) */
static int32_t select_quality(const oracle_scenario *sc, double level, int32_t cur, int has_est, double est) {
    if (level < sc->panic) return 1;
    if (level < sc->safe) return cur - 1 > 1 ? cur - 1 : 1;
    if (cur < sc->n_ranks && has_est && est >= (double)sc->bitrates[cur] * sc->headroom) return cur + 1;
    return cur;
}

/* BandwidthTrace._drain_from (netem.py:77-95) */
static void drain_from(const client_t *c, const double *values, double phase, double bits,
                       double *spent_out, double *left_out) {
    const double *st = c->starts;
    int32_t n = c->n_samples;
    int32_t lo = 0, hi = n;              /* bisect_right */
    while (lo < hi) { int32_t mid = (lo + hi) / 2; if (phase < st[mid]) hi = mid; else lo = mid + 1; }
    int32_t i = lo - 1;
    if (i < 0) i = 0;
    double spent = 0.0, pos = phase;
    for (; i < n; i++) {
        double seg_end = (i + 1 < n) ? st[i + 1] : c->period;
        double width = seg_end - pos;
        if (width > 0) {
            double v = values[i];
            if (v > 0) {
                if (v * width >= bits) { *spent_out = spent + bits / v; *left_out = 0.0; return; }
                bits -= v * width;
            }
            spent += width;
            pos = seg_end;
        }
    }
    *spent_out = spent;
    *left_out = bits;
}

/* BandwidthTrace.completion_time, looping (netem.py:97-118) */
static double completion_time(const world_t *w, const client_t *c, double start, int64_t nbytes) {
    double bits = (double)nbytes * 8.0;
    if (bits <= 0) return start;
    if (c->pbits <= 0) return INFINITY;
    double t = start, spent, left;
    drain_from(c, c->values, fmod(start, c->period), bits, &spent, &left);
    t += spent;
    if (left <= 0) return t;
    double whole = floor(left / c->pbits);
    t += whole * c->period;
    left -= whole * c->pbits;
    if (left <= 0) return t;
    drain_from(c, c->values, 0.0, left, &spent, &left);
    return t + spent;
}

/* ---- client coroutine: client_proc + run_session + InProcessEndpoint ---- */
static void client_step(world_t *w, int32_t cid) {
    const oracle_scenario *sc = w->sc;
    oracle_outputs *o = w->out;
    client_t *c = &w->cl[cid];
    int32_t task = w->n_workers + cid;
    int hung = 0;
    for (;;) {
        switch (c->pc) {
        case C_START: /* await loop.sleep(offsets[cid]) (orchestrator.py:337) */
            c->pc = C_ARRIVED;
            if (do_sleep(w, task, w->arrivals[cid], &hung)) { if (hung) c->pc = C_HUNG; return; }
            break;
        case C_ARRIVED: { /* trace_for + picks stream (orchestrator.py:338-340) */
            uint32_t ent[8]; int m = 0;
            m = push_words(ent, m, sc->seed);
            m = push_words(ent, m, 3);
            m = push_words(ent, m, (uint64_t)cid);
            seed_pcg64(&c->picks, ent, m);
            c->pc = C_SESSION;
            break;
        }
        case C_SESSION: { /* while now < horizon: pick, run_session (orchestrator.py:341-345) */
            if (!(w->now < sc->horizon)) { c->pc = C_DONE; return; }
            int32_t seq;
            if (sc->popularity == POP_ZIPF) {
                double u = pcg_next_double(&c->picks);
                seq = sc->n_seq - 1;
                for (int32_t k = 0; k < sc->n_seq; k++) if (u < sc->zipf_cdf[k]) { seq = k; break; }
            } else {
                seq = (int32_t)pcg_integers(&c->picks, sc->n_seq);
            }
            c->seq = seq;
            int64_t s = o->n_sess++;
            c->session = (int32_t)s;
            c->buf_live = 0;
            if (s < o->sess_cap) {
                o->sess_client[s] = cid; o->sess_seq[s] = seq; o->sess_start[s] = w->now;
                o->sess_end[s] = 0.0; o->sess_stalls[s] = 0; o->sess_stall_time[s] = 0.0;
                o->sess_startup[s] = NAN; o->sess_flags[s] = 0;
            } else {
                set_overflow(w);
            }
            /* endpoint.manifest -> shaped_download (client.py:213-216, netem.py:133-142) */
            c->pc = C_MAN_LAT;
            if (sc->latency > 0) {
                if (do_sleep(w, task, sc->latency, &hung)) { if (hung) c->pc = C_HUNG; return; }
            }
            break;
        }
        case C_MAN_LAT: {
            double start = w->now;
            double end = completion_time(w, c, start, sc->manifest_bytes[c->seq]);
            c->pc = C_MAN_XFER;
            if (do_sleep(w, task, end - start, &hung)) { if (hung) c->pc = C_HUNG; return; }
            break;
        }
        case C_MAN_XFER: /* PlayerBuffer(now); estimate None; rank 1 (client.py:245-248) */
            c->level = 0.0; c->phase = PH_STARTUP; c->position = 0.0; c->last_sync = w->now;
            c->stall_events = 0; c->stall_time = 0.0; c->started_at = NAN; c->session_start = w->now;
            c->buf_live = 1;
            c->has_est = 0; c->est = 0.0; c->rank = 1; c->index = 0;
            c->pc = C_INDEX_HEAD;
            break;
        case C_INDEX_HEAD: /* client.py:250-256 */
            buf_advance(c, w->now);
            __attribute__((fallthrough));
        case C_TARGET_WAIT:
            if (c->pc == C_TARGET_WAIT) buf_advance(c, w->now);
            if (c->phase == PH_PLAYING && c->level >= sc->target) {
                c->pc = C_TARGET_WAIT;
                if (do_sleep(w, task, c->level - sc->target + 1e-9, &hung)) { if (hung) c->pc = C_HUNG; return; }
                break;
            }
            if (c->index > 0) c->rank = select_quality(sc, c->level, c->rank, c->has_est, c->est);
            c->attempt = 0;                  /* _fetch_with_retry (client.py:291-305) */
            c->backoff = sc->retry_backoff;
            /* InProcessEndpoint.segment (client.py:218-226) */
            c->requested = w->now;
            c->pc = C_SEG_LAT;
            if (sc->latency > 0) {
                if (do_sleep(w, task, sc->latency, &hung)) { if (hung) c->pc = C_HUNG; return; }
            }
            break;
        case C_SEG_LAT: { /* MediaServer.segment (server.py:61-78) + Backend.handle (backend.py:115-133) */
            c->req_id = w->req_counter++;
            c->arrival = w->now;
            int32_t d = desc_id(w, c->seq, c->rank, c->index);
            c->desc = d;
            c->size = w->sizes[d];
            if (is_stored(w, c->rank)) {
                c->path = PATH_STORAGE;
            } else {
                if (sc->cache_enabled && cache_get(w, d)) {
                    maybe_speculate(w, c->seq, c->rank, c->index);
                    c->path = PATH_CACHE;
                } else if (w->inflight[d]) {
                    maybe_speculate(w, c->seq, c->rank, c->index);
                    c->path = PATH_WAITED;
                    add_waiter(w, d, cid);
                    c->pc = C_SEG_WAIT;
                    return;
                } else if (enqueue_job(w, d, ORIGIN_DEMAND)) {
                    /* OverloadError: the server records an error (server.py:70-73), the
                     * client backs off or gives up (client.py:291-305, 257-260) */
                    c->path = PATH_ERROR;
                    int64_t sz = c->size;
                    c->size = 0;
                    append_request(w, c, w->now);
                    c->size = sz;
                    if (c->attempt == sc->retries) {
                        if (c->session < o->sess_cap) o->sess_flags[c->session] |= SESS_ABORTED;
                        sync_report(w, c, w->now);
                        c->buf_live = 0;
                        c->pc = C_SESSION;
                        break;
                    }
                    c->pc = C_RETRY;
                    if (do_sleep(w, task, c->backoff, &hung)) { if (hung) c->pc = C_HUNG; return; }
                    break;
                } else {
                    maybe_speculate(w, c->seq, c->rank, c->index);
                    c->path = PATH_TRANSCODED;
                    add_waiter(w, d, cid);
                    c->pc = C_SEG_WAIT;
                    return;
                }
            }
        }
            /* answered without waiting */
            __attribute__((fallthrough));
        case C_SEG_WAIT: {
            append_request(w, c, w->now);
            double start = w->now;
            c->xfer_start = start;
            double end = completion_time(w, c, start, c->size);
            c->pc = C_SEG_XFER;
            if (do_sleep(w, task, end - start, &hung)) { if (hung) c->pc = C_HUNG; return; }
            break;
        }
        case C_SEG_XFER: { /* client.py:261-267 */
            double dt = w->now - c->xfer_start;
            double rate = dt > 0 ? ((double)c->size * 8.0) / dt : INFINITY;
            if (!c->has_est) { c->est = rate; c->has_est = 1; }
            else c->est = sc->alpha * rate + (1.0 - sc->alpha) * c->est;
            double segdur = sc->seq_segdur[c->seq];
            double rem = sc->seq_duration[c->seq] - (double)c->index * segdur;
            double duration = rem < segdur ? rem : segdur;
            buf_on_segment(sc, c, w->now, duration);
            int64_t g = o->n_seg++;
            if (g < o->seg_cap) {
                o->seg_session[g] = c->session; o->seg_index[g] = c->index; o->seg_rep[g] = c->rank;
                o->seg_start[g] = c->requested; o->seg_end[g] = w->now;
            } else {
                set_overflow(w);
            }
            sync_report(w, c, w->now);
            c->index++;
            if (c->index < w->seg_count[c->seq]) { c->pc = C_INDEX_HEAD; break; }
            /* session tail: advance; sleep(level) (client.py:269-271) */
            buf_advance(c, w->now);
            c->pc = C_PLAYOUT;
            if (do_sleep(w, task, c->level, &hung)) { if (hung) c->pc = C_HUNG; return; }
            break;
        }
        case C_RETRY:                        /* after sleep(backoff): backoff *= 2, next attempt */
            c->backoff *= 2.0;
            c->attempt++;
            c->requested = w->now;
            c->pc = C_SEG_LAT;
            if (sc->latency > 0) {
                if (do_sleep(w, task, sc->latency, &hung)) { if (hung) c->pc = C_HUNG; return; }
            }
            break;
        case C_PLAYOUT: /* client.py:272-280 */
            buf_advance(c, w->now);
            c->phase = PH_FINISHED;
            if (c->session < o->sess_cap) o->sess_flags[c->session] |= SESS_FINISHED;
            sync_report(w, c, w->now);
            c->buf_live = 0;
            c->pc = C_SESSION;
            break;
        default:
            return;
        }
    }
}

/* ---- worker coroutine: Backend._worker_loop (backend.py:186-207) ---- */
static void worker_step(world_t *w, int32_t wid, int64_t value) {
    const oracle_scenario *sc = w->sc;
    oracle_outputs *o = w->out;
    worker_t *k = &w->wk[wid];
    int32_t job = (int32_t)value;
    for (;;) {
        switch (k->pc) {
        case W_WOKEN:
        case W_START:
        case W_NEXT:
            if (sc->demand_priority) {       /* Backend._next_job, priority mode (backend.py:174-184) */
                if (w->jq_n > 0) {
                    job = w->jq[w->jq_head]; w->jq_head = (w->jq_head + 1) % w->jq_cap; w->jq_n--;
                    k->pc = W_GOT;
                    break;
                }
                if (w->sq_n > 0) {
                    job = w->sq[w->sq_head]; w->sq_head = (w->sq_head + 1) % w->jq_cap; w->sq_n--;
                    k->pc = W_GOT;
                    break;
                }
                if (w->tokens > 0) { w->tokens--; k->pc = W_NEXT; break; }   /* stale wakeup: no yield */
                w->gq[(w->gq_head + w->gq_n) % w->n_workers] = wid;
                w->gq_n++;
                k->pc = W_WOKEN;
                return;
            }
            if (w->jq_n > 0) { /* Queue.get on a non-empty queue does not yield */
                job = w->jq[w->jq_head];
                w->jq_head = (w->jq_head + 1) % w->jq_cap;
                w->jq_n--;
                k->pc = W_GOT;
                break;
            }
            w->gq[(w->gq_head + w->gq_n) % w->n_workers] = wid;
            w->gq_n++;
            k->pc = W_GOT;
            return;
        case W_GOT: {
            k->job = job;
            if (job >= o->job_cap) { set_overflow(w); k->pc = W_NEXT; return; }
            int32_t d = desc_id(w, o->job_seq[job], o->job_rep[job], o->job_index[job]);
            if (sc->cache_enabled && w->present[d]) {
                o->job_outcome[job] = OUT_DROPPED;
                o->stats[ST_WASTED]++;
                resolve(w, d);
                k->pc = W_NEXT;
                break;
            }
            /* run_transcode (transcode.py:123-128) + ServiceSampler (transcode.py:95-99) */
            o->job_start[job] = w->now;
            int32_t rank = o->job_rep[job];
            double segdur = sc->seq_segdur[o->job_seq[job]];
            double rem = sc->seq_duration[o->job_seq[job]] - (double)o->job_index[job] * segdur;
            double duration = rem < segdur ? rem : segdur;
            double eps = 0.0;
            if (sc->noise > 0) {
                if (k->eps_pos >= sc->eps_per_worker) { set_overflow(w); eps = 0.0; }
                else eps = sc->eps[(int64_t)wid * sc->eps_per_worker + k->eps_pos];
                k->eps_pos++;
            }
            double svc = sc->rho[rank - 1] * duration * (1.0 + eps);
            if (1e-9 > svc) svc = 1e-9;
            heap_push(w, w->now + svc, wid);
            k->pc = W_SERVICE;
            return;
        }
        case W_SERVICE: {
            int32_t j = k->job;
            o->job_fin[j] = w->now;
            o->job_outcome[j] = OUT_COMPLETED;
            int32_t d = desc_id(w, o->job_seq[j], o->job_rep[j], o->job_index[j]);
            if (sc->cache_enabled) cache_put(w, d);
            resolve(w, d);
            k->pc = W_NEXT;
            break;
        }
        default:
            return;
        }
    }
}

static void run_ready(world_t *w) {
    while (w->rq_n > 0) {
        ready_ent e = w->ready[w->rq_head];
        w->rq_head = (w->rq_head + 1) % w->rq_cap;
        w->rq_n--;
        w->out->stats[ST_READY_CALLBACKS]++;
        if (e.task < w->n_workers) worker_step(w, e.task, e.value);
        else client_step(w, e.task - w->n_workers);
    }
}

/* ------------------------------------------------------------------------ */
/* Public entry points.                                                     */
/* ------------------------------------------------------------------------ */

int oracle_segment_sizes(const oracle_scenario *sc, int64_t *sizes, int32_t *counts) {
    /* Catalog.segment_count / descriptor (content.py:204-218) */
    for (int32_t s = 0; s < sc->n_seq; s++) {
        double q = sc->seq_duration[s] / sc->seq_segdur[s];
        counts[s] = (int32_t)ceil(q);
    }
    for (int32_t s = 0; s < sc->n_seq; s++)
        for (int32_t r = 1; r <= sc->n_ranks; r++)
            for (int32_t i = 0; i < sc->max_nseg; i++) {
                int64_t *dst = &sizes[((int64_t)s * sc->n_ranks + (r - 1)) * sc->max_nseg + i];
                if (i >= counts[s]) { *dst = 0; continue; }
                double segdur = sc->seq_segdur[s];
                double rem = sc->seq_duration[s] - (double)i * segdur;
                double duration = rem < segdur ? rem : segdur;
                double base = ((double)sc->bitrates[r - 1] * duration) / 8.0;
                uint32_t ent[16]; int m = 0;
                m = push_words(ent, m, sc->catalog_seed);
                m = push_words(ent, m, (uint64_t)sc->seq_key[s]);
                m = push_words(ent, m, (uint64_t)r);
                m = push_words(ent, m, (uint64_t)i);
                pcg64_t g;
                seed_pcg64(&g, ent, m);
                double j = sc->size_jitter;
                double u = -j + (j - -j) * pcg_next_double(&g);
                double v = nearbyint(base * (1.0 + u));   /* round(): half-even */
                int64_t size = (int64_t)v;
                *dst = size > 1 ? size : 1;
            }
    return 0;
}

int oracle_build_traces(const oracle_scenario *sc, double *values, double *pbits, double *period) {
    int32_t n = sc->n_samples;
    double *ts = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_sample_times(sc->trace_duration, sc->trace_step, ts, n);
    for (int32_t c = 0; c < sc->n_clients; c++)
        build_trace(sc, sc->trace_normals + (int64_t)c * (n + 1), ts, n,
                    values + (int64_t)c * n, period, &pbits[c]);
    free(ts);
    return 0;
}

int oracle_run(const oracle_scenario *sc, oracle_outputs *out) {
    world_t W;
    memset(&W, 0, sizeof W);
    world_t *w = &W;
    w->sc = sc;
    w->out = out;
    out->n_req = out->n_sess = out->n_seg = out->n_job = 0;
    memset(out->stats, 0, sizeof out->stats);
    w->n_clients = sc->n_clients;
    w->n_workers = sc->n_workers;
    w->n_tasks = sc->n_clients + sc->n_workers;
    w->n_desc = sc->n_seq * sc->n_ranks * sc->max_nseg;
    w->sizes = (int64_t *)malloc(sizeof(int64_t) * (size_t)w->n_desc);
    w->seg_count = (int32_t *)malloc(sizeof(int32_t) * (size_t)sc->n_seq);
    oracle_segment_sizes(sc, w->sizes, w->seg_count);

    /* traces: synthetic (one per client, timestamps shared) unless CSV tables are given */
    const int csv = sc->tr_off != NULL;
    w->n_samples = csv ? 1 : sc->n_samples;
    double *ts = (double *)malloc(sizeof(double) * (size_t)w->n_samples);
    double *vals = (double *)malloc(sizeof(double) * (size_t)w->n_samples * (size_t)(csv ? 1 : sc->n_clients));
    double *pb = (double *)malloc(sizeof(double) * (size_t)sc->n_clients);
    if (!csv) {
        oracle_sample_times(sc->trace_duration, sc->trace_step, ts, sc->n_samples);
        if (ts[0] > 0) ts[0] = 0.0;
        oracle_build_traces(sc, vals, pb, &w->period);
    }
    w->starts = ts;

    /* arrival offsets: list(np.cumsum(exponential draws)) (orchestrator.py:265-268) */
    double *arr = (double *)malloc(sizeof(double) * (size_t)sc->n_clients);
    double acc = 0.0;
    for (int32_t c = 0; c < sc->n_clients; c++) { acc += sc->arrival_draws[c]; arr[c] = acc; }
    w->arrivals = arr;

    w->cl = (client_t *)calloc((size_t)sc->n_clients, sizeof(client_t));
    w->wk = (worker_t *)calloc((size_t)sc->n_workers, sizeof(worker_t));
    for (int32_t c = 0; c < sc->n_clients; c++) {
        client_t *cl = &w->cl[c];
        if (csv) {
            cl->starts = sc->tr_starts + sc->tr_off[c];
            cl->values = sc->tr_values + sc->tr_off[c];
            cl->n_samples = sc->tr_n[c];
            cl->period = sc->tr_period[c];
            cl->pbits = sc->tr_pbits[c];
        } else {
            cl->starts = ts;
            cl->values = vals + (int64_t)c * sc->n_samples;
            cl->n_samples = sc->n_samples;
            cl->period = w->period;
            cl->pbits = pb[c];
        }
        cl->wait_next = -1;
    }
    w->heap = (timer_ent *)malloc(sizeof(timer_ent) * (size_t)(w->n_tasks + 1));
    w->rq_cap = w->n_tasks + 1;
    w->ready = (ready_ent *)malloc(sizeof(ready_ent) * (size_t)w->rq_cap);
    w->present = (int8_t *)calloc((size_t)w->n_desc, 1);
    w->inflight = (int8_t *)calloc((size_t)w->n_desc, 1);
    w->lru_prev = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->n_desc);
    w->lru_next = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->n_desc);
    w->wq_head = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->n_desc);
    w->wq_tail = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->n_desc);
    w->lru_head = w->lru_tail = -1;
    w->jq_cap = w->n_desc + 1;   /* single-flight: <= one queued job per descriptor */
    w->jq = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->jq_cap);
    w->gq = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->n_workers);
    w->sq = (int32_t *)malloc(sizeof(int32_t) * (size_t)w->jq_cap);

    /* spawn order: K workers (backend.py:110) then N clients (orchestrator.py:350-351) */
    for (int32_t k = 0; k < w->n_workers; k++) ready_push(w, k, 0);
    for (int32_t c = 0; c < w->n_clients; c++) ready_push(w, w->n_workers + c, 0);
    w->now = 0.0;

    /* VirtualLoop.run_until(horizon) (sim.py:347-360) */
    run_ready(w);
    while (w->heap_n > 0 && w->heap[0].when <= sc->horizon) {
        timer_ent e = heap_pop(w);
        w->now = e.when;
        out->stats[ST_TIMER_POPS]++;
        ready_push(w, e.task, 0);   /* fut.set_result -> call_soon(task._resume) */
        run_ready(w);
        if (w->status) break;
    }
    if (sc->horizon > w->now) w->now = sc->horizon;

    /* harvest (orchestrator.py:357-359, client.py:177-187) */
    for (int32_t c = 0; c < w->n_clients; c++) {
        client_t *cl = &w->cl[c];
        if (cl->buf_live && cl->pc != C_DONE) {
            buf_advance(cl, w->now);
            sync_report(w, cl, w->now);
        }
        if (cl->pc == C_HUNG) out->stats[ST_HUNG]++;
    }

    out->stats[ST_CACHE_CAPACITY] = sc->cache_capacity;
    out->stats[ST_CURRENT_BYTES] = w->cur_bytes;
    out->stats[ST_ENTRIES] = w->entries;
    out->stats[ST_STATUS] = w->status;

    free(w->sizes); free(w->seg_count); free(ts); free(vals); free(pb);
    free(w->cl); free(w->wk); free(w->heap); free(w->ready);
    free(w->present); free(w->inflight); free(w->lru_prev); free(w->lru_next);
    free(w->wq_head); free(w->wq_tail); free(w->jq); free(w->gq); free(w->sq); free(arr);
    return w->status;
}

int oracle_libm(int fn, const double *x, int64_t n, double *out) {
    if (fn != 0 && fn != 1) return 1;
    for (int64_t i = 0; i < n; i++) out[i] = fn == 0 ? exp(x[i]) : log1p(x[i]);
    return 0;
}
