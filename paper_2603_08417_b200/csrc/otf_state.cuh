// otf_state.cuh -- per-scenario engine state (lives in the scratch arena).
#pragma once
#include <stdint.h>

#include "otf_model.cuh"
#include "otf_rng.cuh"
#include "otf_xacc.cuh"
#include "otfgpu.h"

namespace otf {

// Client coroutine program counter: where client_proc/run_session is parked
// (orchestrator.py:336-348, client.py:229-305, netem.py:133-142).
enum {
    C_START = 0,    // spawned; next: sleep(offset)
    C_ARRIVED,      // woke from the arrival sleep
    C_SESSION,      // top of `while now < horizon`
    C_MAN_LAT,      // manifest latency sleep
    C_MAN_XFER,     // manifest shaped transfer
    C_INDEX_HEAD,   // top of the per-segment loop
    C_TARGET_WAIT,  // buffer-full wait (client.py:252-254)
    C_SEG_LAT,      // request latency sleep -> MediaServer.segment on wake
    C_SEG_WAIT,     // awaiting a transcode waiter Future
    C_SEG_RESP,     // response available (windowed engine): record + transfer
    C_SEG_XFER,     // shaped segment transfer
    C_PLAYOUT,      // final sleep(level)
    C_SEG_ERR,      // OverloadError response (windowed engine): record, then retry or abort
    C_RETRY,        // sleep(backoff) before the next attempt (client.py:297-300)
    C_DONE,         // client_proc returned (now >= horizon)
    C_HUNG          // slept on an infinite delay; never wakes
};

struct Client {                 // 144 B: moved as a whole per event
    Buffer buf;                 // 48 B
    double est, requested, arrival, xfer_start;
    double next_when, ctime;    // windowed engine: pending timer (fire time, arm time)
    int32_t req_id, size, req_slot;
    int32_t pc, seq, session, index, rank;
    int32_t path, desc, wait_next;
    uint8_t has_est, buf_live, sess_open;
    uint8_t attempt;            // _fetch_with_retry attempt (client.py:291-305); the backoff is
                                // retry_backoff_s * 2^attempt (repeated doubling is exact)
};                              // the pick stream lives in a separate (cold) array

// The per-client state touched only at session boundaries: the sequence-pick
// stream (orchestrator.py:338-342) and the session's registration time (the
// order the reference sums stall times in, metrics.py:88-92).
struct ClientCold {              // 64 B
    Pcg64 picks;
    double reg_time;
    double pad;
};

// QoE accumulators while a scenario runs: 32-bit counters (native shared /
// global atomics) and the summary-tail cursors.  Session-level numbers are
// not counted here: a closing session appends its record (otf_sess_ent) and
// the summary pass derives the session histograms and sums (otf_summary.cu).
struct QoeAcc {
    uint32_t lat_hist[OTF_LAT_BINS];
    uint32_t path_count[8];             // n_requests = their sum
    uint32_t rank_count[OTF_RANK_BINS];
    uint32_t n_segments;
    uint32_t n_lat_tail, n_ses_tail, n_sup_tail;   // tail cursors (exact counts, even past a cap)
    uint32_t flags, pad[3];
};

enum { W_START = 0, W_NEXT, W_GOT, W_SERVICE, W_WOKEN };

struct Worker {
    int32_t pc, desc, job, pad;
    int64_t eps_pos;
};

struct Desc {                   // per (seq, rank, index) descriptor
    int32_t lru_prev, lru_next; // SegmentCache OrderedDict order (cache.py:27-92)
    int32_t wq_head, wq_tail;   // in-flight waiter Future callbacks, await order
    int32_t flags;              // bit0 cached, bit1 in-flight
};
enum { D_CACHED = 1, D_INFLIGHT = 2 };

struct Timer {
    double when;
    uint32_t tick;
    int32_t task;
};

struct ReadyEnt {
    int32_t task, desc, job, pad;
};

struct JobEnt {
    int32_t desc, job;
};

OTF_HD int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

struct ExactLayout {
    int64_t state, clients, picks, workers, heap, ready, descs, jobq, specq, getq, total;
};

OTF_HD ExactLayout exact_layout(int32_t n_clients, int32_t n_workers, int64_t n_desc) {
    ExactLayout L;
    int64_t n_tasks = (int64_t)n_clients + n_workers;
    int64_t o = 0;
    L.state = o; o += 256;                     // EngineState
    o += align256(sizeof(QoeAcc));             // QoeAcc (at state + 256)
    L.clients = o; o += align256((int64_t)sizeof(Client) * n_clients);
    L.picks = o;   o += align256((int64_t)sizeof(ClientCold) * n_clients);
    L.workers = o; o += align256((int64_t)sizeof(Worker) * n_workers);
    L.heap = o;    o += align256((int64_t)sizeof(Timer) * (n_tasks + 1));
    L.ready = o;   o += align256((int64_t)sizeof(ReadyEnt) * (n_tasks + 1));
    L.descs = o;   o += align256((int64_t)sizeof(Desc) * n_desc);
    L.jobq = o;    o += align256((int64_t)sizeof(JobEnt) * (n_desc + 1));
    L.specq = o;   o += align256((int64_t)sizeof(JobEnt) * (n_desc + 1));
    L.getq = o;    o += align256((int64_t)sizeof(int32_t) * n_workers);
    L.total = o;
    return L;
}

}  // namespace otf
