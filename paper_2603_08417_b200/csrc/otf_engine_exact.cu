// otf_engine_exact.cu -- the exact engine: one thread replays one scenario.
//
// A literal device-side replay of VirtualLoop.run_until (sim.py:347-360): a
// binary min-heap of (when, tick) timers, a FIFO ready ring drained after
// every timer pop, and explicit state machines for the client coroutines
// (orchestrator.py:336-348 + client.py:229-305) and the K transcode workers
// (backend.py:186-216).  It reproduces every tie-break of the reference
// (tick order, ready-queue hop, getter FIFO, waiter callback order), so it is
// the ground truth the windowed engine falls back to when it meets a tie it
// cannot order.  All state lives in the scenario's scratch arena.
#include <math.h>
#include <stdint.h>

#include "otf_engine_common.cuh"

namespace otf {

struct ExactWorld {
    Scn S;                  // scenario view (tables, outputs, counters)
    Client *cl;
    Worker *wk;
    Timer *heap;
    ReadyEnt *ready;
    Desc *descs;
    JobEnt *jq, *sq;                        // demand / speculative job FIFOs
    int32_t *gq;
    int32_t heap_n, rq_head, rq_n, rq_cap;
    int32_t jq_head, jq_n, jq_cap, gq_head, gq_n;
    int32_t sq_head, sq_n, tokens;          // demand-priority mode (backend.py:103-105)
    uint32_t tick;
    double now;
};

__device__ __forceinline__ bool tm_less(const Timer &a, const Timer &b) {
    return a.when < b.when || (a.when == b.when && a.tick < b.tick);
}

// VirtualLoop.call_at (sim.py:304-309)
__device__ void heap_push(ExactWorld &w, double when, int32_t task) {
    int32_t i = w.heap_n++;
    Timer e;
    e.when = when; e.tick = w.tick++; e.task = task;
    if (w.tick == 0) w.S.flag(OTF_S_INTERNAL);   // tick wrapped
    while (i > 0) {
        int32_t p = (i - 1) >> 1;
        Timer tp = w.heap[p];
        if (!tm_less(e, tp)) break;
        w.heap[i] = tp;
        i = p;
    }
    w.heap[i] = e;
}

__device__ Timer heap_pop(ExactWorld &w) {
    Timer top = w.heap[0];
    Timer last = w.heap[--w.heap_n];
    int32_t i = 0, n = w.heap_n;
    for (;;) {
        int32_t l = 2 * i + 1, r = l + 1, m = i;
        Timer best = last;
        if (l < n) { Timer tl = w.heap[l]; if (tm_less(tl, best)) { m = l; best = tl; } }
        if (r < n) { Timer tr = w.heap[r]; if (tm_less(tr, best)) { m = r; best = tr; } }
        if (m == i) break;
        w.heap[i] = best;
        i = m;
    }
    if (n > 0) w.heap[i] = last;
    return top;
}

__device__ __forceinline__ void ready_push(ExactWorld &w, int32_t task, int32_t desc, int32_t job) {
    int32_t pos = w.rq_head + w.rq_n;
    if (pos >= w.rq_cap) pos -= w.rq_cap;
    ReadyEnt e; e.task = task; e.desc = desc; e.job = job; e.pad = 0;
    w.ready[pos] = e;
    w.rq_n++;
}

// loop.sleep(delay) (sim.py:317-324); true when the coroutine yields.
__device__ __forceinline__ bool do_sleep(ExactWorld &w, Client &c, int32_t task, double delay) {
    if (delay <= 0) return false;
    if (isinf(delay)) { c.pc = C_HUNG; return true; }
    heap_push(w, w.now + delay, task);
    return true;
}

// ---- cache (cache.py:45-81) --------------------------------------------------
__device__ void lru_unlink(ExactWorld &w, int32_t d) {
    Desc &D = w.descs[d];
    int32_t p = D.lru_prev, n = D.lru_next;
    if (p >= 0) w.descs[p].lru_next = n; else w.S.st->lru_head = n;
    if (n >= 0) w.descs[n].lru_prev = p; else w.S.st->lru_tail = p;
}
__device__ void lru_append(ExactWorld &w, int32_t d) {
    int32_t t = w.S.st->lru_tail;
    w.descs[d].lru_prev = t;
    w.descs[d].lru_next = -1;
    if (t >= 0) w.descs[t].lru_next = d; else w.S.st->lru_head = d;
    w.S.st->lru_tail = d;
}
__device__ bool cache_get(ExactWorld &w, int32_t d) {
    if (!(w.descs[d].flags & D_CACHED)) { w.S.stat(OTF_ST_MISSES)++; return false; }
    lru_unlink(w, d);
    lru_append(w, d);
    w.S.stat(OTF_ST_HITS)++;
    return true;
}
__device__ void cache_put(ExactWorld &w, int32_t d) {
    int64_t size = w.S.size(d);
    int64_t cap = w.S.sc->cache_capacity;
    EngineState *st = w.S.st;
    if (size > cap) { w.S.stat(OTF_ST_REJECTED)++; return; }
    if (w.descs[d].flags & D_CACHED) {
        st->cur_bytes -= size;
        lru_unlink(w, d);
        w.descs[d].flags &= ~D_CACHED;
        st->entries--;
    }
    while (st->cur_bytes + size > cap) {
        int32_t v = st->lru_head;
        lru_unlink(w, v);
        w.descs[v].flags &= ~D_CACHED;
        st->entries--;
        st->cur_bytes -= w.S.size(v);
        w.S.stat(OTF_ST_EVICTIONS)++;
    }
    lru_append(w, d);
    w.descs[d].flags |= D_CACHED;
    st->entries++;
    st->cur_bytes += size;
}

// ---- backend (backend.py:135-216) --------------------------------------------
// Backend._enqueue + Queue.put_nowait (backend.py:156-170, sim.py:229-240).
// Returns true on OverloadError: no idle worker and the queue at its bound.
__device__ bool enqueue_job(ExactWorld &w, int32_t d, int32_t origin) {
    const bool prio = w.S.sc->demand_priority != 0;
    if (prio) {                             // workers never wait on the job queues in this mode
        if (origin == OTF_ORIGIN_DEMAND && w.S.sc->queue_bound > 0 && w.jq_n >= w.S.sc->queue_bound) return true;
    } else if (w.gq_n == 0 && w.S.sc->queue_bound > 0 && w.jq_n >= w.S.sc->queue_bound) {
        return true;
    }
    int32_t j = w.S.record_job(d, origin, w.now);
    Desc &D = w.descs[d];
    D.flags |= D_INFLIGHT;
    D.wq_head = D.wq_tail = -1;
    if (prio) {                             // separate FIFOs + _wakeup.put_nowait(None, force=True)
        JobEnt e; e.desc = d; e.job = j;
        if (origin == OTF_ORIGIN_SPECULATIVE) {
            int32_t pos = w.sq_head + w.sq_n; if (pos >= w.jq_cap) pos -= w.jq_cap;
            w.sq[pos] = e; w.sq_n++;
        } else {
            int32_t pos = w.jq_head + w.jq_n; if (pos >= w.jq_cap) pos -= w.jq_cap;
            w.jq[pos] = e; w.jq_n++;
        }
        if (w.gq_n > 0) {
            int32_t wid = w.gq[w.gq_head];
            w.gq_head = (w.gq_head + 1 == w.S.sc->n_workers) ? 0 : w.gq_head + 1;
            w.gq_n--;
            ready_push(w, wid, -1, -1);
        } else {
            w.tokens++;
        }
        return false;
    }
    if (w.gq_n > 0) {                         // hand to the first waiting getter
        int32_t wid = w.gq[w.gq_head];
        w.gq_head = (w.gq_head + 1 == w.S.sc->n_workers) ? 0 : w.gq_head + 1;
        w.gq_n--;
        ready_push(w, wid, d, j);
    } else {
        if (w.jq_n >= w.jq_cap) { w.S.flag(OTF_S_INTERNAL); return false; }
        int32_t pos = w.jq_head + w.jq_n;
        if (pos >= w.jq_cap) pos -= w.jq_cap;
        JobEnt e; e.desc = d; e.job = j;
        w.jq[pos] = e;
        w.jq_n++;
    }
    return false;
}

// Backend.maybe_speculate (backend.py:135-154)
__device__ void maybe_speculate(ExactWorld &w, int32_t seq, int32_t rank, int32_t index) {
    if (!w.S.sc->spec_enabled) { w.S.stat(OTF_ST_SKIP_DISABLED)++; return; }
    int32_t ni = index + 1;
    if (ni >= w.S.segcount(seq)) { w.S.stat(OTF_ST_SKIP_EOS)++; return; }
    if (w.S.stored(rank)) { w.S.stat(OTF_ST_SKIP_STORED)++; return; }
    int32_t d = w.S.desc_id(seq, rank, ni);
    int32_t f = w.descs[d].flags;
    if (w.S.sc->cache_enabled && (f & D_CACHED)) { w.S.stat(OTF_ST_SKIP_CACHED)++; return; }
    if (f & D_INFLIGHT) { w.S.stat(OTF_ST_SKIP_INFLIGHT)++; return; }
    if (enqueue_job(w, d, OTF_ORIGIN_SPECULATIVE)) { w.S.stat(OTF_ST_SKIP_OVERLOAD)++; return; }
    w.S.stat(OTF_ST_SPEC_ENQUEUED)++;
}

// Backend._resolve (backend.py:209-216): waiter callbacks in await order.
__device__ void resolve(ExactWorld &w, int32_t d) {
    Desc &D = w.descs[d];
    if (!(D.flags & D_INFLIGHT)) return;
    D.flags &= ~D_INFLIGHT;
    for (int32_t c = D.wq_head; c >= 0; c = w.cl[c].wait_next)
        ready_push(w, w.S.sc->n_workers + c, 0, 0);
    D.wq_head = D.wq_tail = -1;
}

__device__ void add_waiter(ExactWorld &w, int32_t d, int32_t cid) {
    Desc &D = w.descs[d];
    w.cl[cid].wait_next = -1;
    if (D.wq_tail >= 0) w.cl[D.wq_tail].wait_next = cid; else D.wq_head = cid;
    D.wq_tail = cid;
}

// ---- client coroutine ---------------------------------------------------------
__device__ void client_step(ExactWorld &w, int32_t cid) {
    const otf_scenario &sc = *w.S.sc;
    Client &c = w.cl[cid];
    const int32_t task = sc.n_workers + cid;
    for (;;) {
        switch (c.pc) {
        case C_START:                       // await loop.sleep(offsets[cid]) (orchestrator.py:337)
            c.pc = C_ARRIVED;
            if (do_sleep(w, c, task, w.S.arrival(cid))) return;
            break;
        case C_ARRIVED:                     // picks = PCG64(SS([seed, 3, cid])) (orchestrator.py:340)
            client_arrive(w.S, c, cid);
            c.pc = C_SESSION;
            break;
        case C_SESSION:                     // while now < horizon: pick + run_session
            if (!(w.now < sc.horizon)) { c.pc = C_DONE; return; }
            client_new_session(w.S, c, cid, w.now);
            c.pc = C_MAN_LAT;
            if (sc.latency > 0 && do_sleep(w, c, task, sc.latency)) return;
            break;
        case C_MAN_LAT: {                   // shaped manifest transfer (netem.py:133-142)
            double start = w.now;
            double end = completion_time(w.S.trace(cid), start, w.S.manifest(c.seq));
            c.pc = C_MAN_XFER;
            if (do_sleep(w, c, task, end - start)) return;
            break;
        }
        case C_MAN_XFER:                    // PlayerBuffer(now); estimate None; rank 1
            client_start_playback(c, w.now);
            c.pc = C_INDEX_HEAD;
            break;
        case C_INDEX_HEAD:
        case C_TARGET_WAIT:                 // client.py:251-256
            buf_advance(c.buf, w.now);
            if (c.buf.phase == PH_PLAYING && c.buf.level >= sc.target) {
                c.pc = C_TARGET_WAIT;
                if (do_sleep(w, c, task, c.buf.level - sc.target + 1e-9)) return;
                break;
            }
            client_select(w.S, c);
            c.attempt = 0;                  // _fetch_with_retry (client.py:291-305)
            c.requested = w.now;            // InProcessEndpoint.segment (client.py:219-221)
            c.pc = C_SEG_LAT;
            if (sc.latency > 0 && do_sleep(w, c, task, sc.latency)) return;
            break;
        case C_SEG_LAT: {                   // MediaServer.segment + Backend.handle
            c.req_id = (int32_t)w.S.st->req_counter++;
            c.arrival = w.now;
            int32_t d = w.S.desc_id(c.seq, c.rank, c.index);
            c.desc = d;
            c.size = (int32_t)w.S.size(d);
            c.pc = C_SEG_WAIT;
            if (w.S.stored(c.rank)) {
                c.path = OTF_PATH_STORAGE;
            } else if (sc.cache_enabled && cache_get(w, d)) {
                maybe_speculate(w, c.seq, c.rank, c.index);
                c.path = OTF_PATH_CACHE;
            } else if (w.descs[d].flags & D_INFLIGHT) {
                maybe_speculate(w, c.seq, c.rank, c.index);
                c.path = OTF_PATH_WAITED;
                add_waiter(w, d, cid);
                return;
            } else if (enqueue_job(w, d, OTF_ORIGIN_DEMAND)) {
                // OverloadError: error record (server.py:70-73), then retry or give up
                c.path = OTF_PATH_ERROR;
                int32_t sz = c.size;
                c.size = 0;
                w.S.record_request(c, w.now);
                c.size = sz;
                if (c.attempt == sc.retries) {
                    client_abort_session(w.S, c, cid, w.now);
                    c.pc = C_SESSION;
                    break;
                }
                c.pc = C_RETRY;
                if (do_sleep(w, c, task, ldexp(sc.retry_backoff, c.attempt))) return;
                break;
            } else {
                maybe_speculate(w, c.seq, c.rank, c.index);
                c.path = OTF_PATH_TRANSCODED;
                add_waiter(w, d, cid);
                return;
            }
            break;                          // answered without yielding
        }
        case C_SEG_WAIT: {                  // response: record, then shaped transfer
            w.S.record_request(c, w.now);
            double start = w.now;
            c.xfer_start = start;
            double end = completion_time(w.S.trace(cid), start, c.size);
            c.pc = C_SEG_XFER;
            if (do_sleep(w, c, task, end - start)) return;
            break;
        }
        case C_SEG_XFER:                    // client.py:261-271
            if (client_segment_done(w.S, c, w.now)) {
                c.pc = C_INDEX_HEAD;
                break;
            }
            c.pc = C_PLAYOUT;
            if (do_sleep(w, c, task, c.buf.level)) return;
            break;
        case C_RETRY:                       // after sleep(backoff): backoff *= 2, next attempt
            c.attempt++;
            c.requested = w.now;
            c.pc = C_SEG_LAT;
            if (sc.latency > 0 && do_sleep(w, c, task, sc.latency)) return;
            break;
        case C_PLAYOUT:                     // client.py:272-280
            client_finish_session(w.S, c, cid, w.now);
            c.pc = C_SESSION;
            break;
        default:
            return;
        }
    }
}

// ---- worker coroutine (backend.py:186-207) -------------------------------------
__device__ void worker_step(ExactWorld &w, int32_t wid, int32_t desc, int32_t job) {
    const otf_scenario &sc = *w.S.sc;
    Worker &k = w.wk[wid];
    for (;;) {
        switch (k.pc) {
        case W_WOKEN:
        case W_START:
        case W_NEXT:
            if (sc.demand_priority) {       // Backend._next_job, priority mode (backend.py:174-184)
                if (w.jq_n > 0 || w.sq_n > 0) {
                    JobEnt e;
                    if (w.jq_n > 0) { e = w.jq[w.jq_head]; w.jq_head = (w.jq_head + 1 == w.jq_cap) ? 0 : w.jq_head + 1; w.jq_n--; }
                    else { e = w.sq[w.sq_head]; w.sq_head = (w.sq_head + 1 == w.jq_cap) ? 0 : w.sq_head + 1; w.sq_n--; }
                    desc = e.desc; job = e.job;
                    k.pc = W_GOT;
                    break;
                }
                if (w.tokens > 0) { w.tokens--; k.pc = W_NEXT; break; }   // stale wakeup: no yield
                int32_t pos = w.gq_head + w.gq_n;
                if (pos >= sc.n_workers) pos -= sc.n_workers;
                w.gq[pos] = wid;
                w.gq_n++;
                k.pc = W_WOKEN;
                return;
            }
            if (w.jq_n > 0) {               // Queue.get on a non-empty queue: no yield
                JobEnt e = w.jq[w.jq_head];
                w.jq_head = (w.jq_head + 1 == w.jq_cap) ? 0 : w.jq_head + 1;
                w.jq_n--;
                desc = e.desc; job = e.job;
                k.pc = W_GOT;
                break;
            }
            {
                int32_t pos = w.gq_head + w.gq_n;
                if (pos >= sc.n_workers) pos -= sc.n_workers;
                w.gq[pos] = wid;
                w.gq_n++;
            }
            k.pc = W_GOT;
            return;
        case W_GOT:
            k.desc = desc; k.job = job;
            if (sc.cache_enabled && (w.descs[desc].flags & D_CACHED)) {   // dedup on dequeue
                w.S.job_outcome(job, OTF_OUTCOME_DROPPED);
                w.S.stat(OTF_ST_WASTED)++;
                resolve(w, desc);
                k.pc = W_NEXT;
                break;
            }
            {                               // run_transcode (transcode.py:123-128)
                w.S.job_started(job, w.now);
                double svc = w.S.service_time(k, wid, desc);
                heap_push(w, w.now + svc, wid);
            }
            k.pc = W_SERVICE;
            return;
        case W_SERVICE:                     // transcode.py:129-131, backend.py:205-207
            w.S.job_finished(job = k.job, w.now);
            if (sc.cache_enabled) cache_put(w, k.desc);
            resolve(w, k.desc);
            k.pc = W_NEXT;
            break;
        default:
            return;
        }
    }
}

__device__ void run_ready(ExactWorld &w) {
    while (w.rq_n > 0) {
        ReadyEnt e = w.ready[w.rq_head];
        w.rq_head = (w.rq_head + 1 == w.rq_cap) ? 0 : w.rq_head + 1;
        w.rq_n--;
        w.S.stat(OTF_ST_READY_CALLBACKS)++;
        if (e.task < w.S.sc->n_workers) worker_step(w, e.task, e.desc, e.job);
        else client_step(w, e.task - w.S.sc->n_workers);
    }
}

__global__ void __launch_bounds__(64) exact_kernel(const otf_batch b) {
    int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b.n_scenarios) return;
    int32_t s = b.order ? b.order[t] : t;
    ExactWorld w;
    otf_batch bl = b;
    w.S.init(&bl, &b.scenarios[s], s);
    w.S.qa = (QoeAcc *)(b.scratch + b.scenarios[s].scratch_off + 256);
    w.S.reset_outputs();
    const otf_scenario &sc = *w.S.sc;
    int64_t n_desc = (int64_t)sc.n_seq * sc.n_ranks * sc.max_nseg;
    ExactLayout L = exact_layout(sc.n_clients, sc.n_workers, n_desc);
    uint8_t *base = b.scratch + sc.scratch_off;
    w.cl = (Client *)(base + L.clients);
    w.S.cold = (ClientCold *)(base + L.picks);
    w.wk = (Worker *)(base + L.workers);
    w.heap = (Timer *)(base + L.heap);
    w.ready = (ReadyEnt *)(base + L.ready);
    w.descs = (Desc *)(base + L.descs);
    w.jq = (JobEnt *)(base + L.jobq);
    w.sq = (JobEnt *)(base + L.specq);
    w.sq_head = 0; w.sq_n = 0; w.tokens = 0;
    w.gq = (int32_t *)(base + L.getq);
    w.heap_n = 0; w.rq_head = 0; w.rq_n = 0;
    w.rq_cap = sc.n_clients + sc.n_workers + 1;
    w.jq_head = 0; w.jq_n = 0; w.jq_cap = (int32_t)(n_desc + 1);
    w.gq_head = 0; w.gq_n = 0;
    w.tick = 0;
    w.now = 0.0;
    for (int64_t d = 0; d < n_desc; d++) {
        Desc D; D.lru_prev = D.lru_next = -1; D.wq_head = D.wq_tail = -1; D.flags = 0;
        w.descs[d] = D;
    }
    for (int32_t c = 0; c < sc.n_clients; c++) client_init(w.cl[c]);
    for (int32_t k = 0; k < sc.n_workers; k++) { Worker K; K.pc = W_START; K.desc = -1; K.job = -1; K.pad = 0; K.eps_pos = 0; w.wk[k] = K; }

    // spawn order: K workers (backend.py:110) then N clients (orchestrator.py:350-351)
    for (int32_t k = 0; k < sc.n_workers; k++) ready_push(w, k, 0, 0);
    for (int32_t c = 0; c < sc.n_clients; c++) ready_push(w, sc.n_workers + c, 0, 0);

    // VirtualLoop.run_until(horizon) (sim.py:347-360)
    run_ready(w);
    while (w.heap_n > 0 && w.heap[0].when <= sc.horizon) {
        Timer e = heap_pop(w);
        w.now = e.when;
        w.S.stat(OTF_ST_TIMER_POPS)++;
        ready_push(w, e.task, 0, 0);     // fut.set_result -> call_soon(task._resume)
        run_ready(w);
        if (w.S.st->status & OTF_S_INTERNAL) break;
    }
    if (sc.horizon > w.now) w.now = sc.horizon;

    // harvest at the horizon (orchestrator.py:357-359, client.py:177-187)
    for (int32_t c = 0; c < sc.n_clients; c++) client_harvest(w.S, w.cl[c], c, w.now);
    w.S.finish();
    w.S.flush_qoe();
}

}  // namespace otf

int otf_launch_exact(const otf_batch &b, cudaStream_t stream) {
    int threads = 32;
    int blocks = (b.n_scenarios + threads - 1) / threads;
    otf::exact_kernel<<<blocks, threads, 0, stream>>>(b);
    return 0;
}
