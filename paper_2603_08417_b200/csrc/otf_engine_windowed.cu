// otf_engine_windowed.cu -- the windowed engine: one warp replays one scenario.
//
// Why it is exact.  In the reference every client->server interaction
// (MediaServer.segment, server.py:61-78) happens when a request-latency timer
// fires, and that timer was armed `latency` seconds earlier
// (InProcessEndpoint.segment, client.py:219-221).  Client-local events
// (manifest transfer, buffer-full waits, segment transfers, play-out,
// session restarts) only touch their own client, and server->client effects
// are responses delivered at the server event's instant.  Cutting virtual time
// into windows [k*W, (k+1)*W) with W slightly below `latency` therefore gives:
//   * every server event of window k was armed before the window started, so
//     the server pass can replay all of them -- plus the worker service timers
//     (backend.py:186-216) and the ready-queue hops they cause (sim.py:126-130,
//     229-247) -- in exact (time, tick) order first.  In request-only windows
//     the whole warp does it (phase_a_parallel: per-(sequence, rank) groups on
//     their owner lanes, sequence numbers by prefix sums); otherwise lane 0;
//   * afterwards the clients just responded to, and the window's local timers,
//     run on the 32 lanes (client.py:229-305, orchestrator.py:336-348).  A
//     client in a local sleep cannot be reached by anyone else, so each runs
//     its local chain in place up to its next request (arm()).
// The only order information this loses is the global tick counter
// (sim.py:304-309), which breaks ties between timers at the identical
// instant.  Server events are ordered by (time, creation time) and ties the
// engine cannot order are flagged (OTF_S_TIE) so the host re-runs that
// scenario on the exact engine; session registration ties are checked on the
// host.  Parity tests pin both engines to the reference's outputs.
//
// Layout: scenario hot state in shared memory (timer-wheel counts and bitmap,
// descriptor words with the waiter-list tails, client links, the window's
// server-event list, worker timers, counters); client coroutine state, the
// wheel's bucket arrays, the job FIFOs and the LRU touch queue in the
// scenario's global scratch arena.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <math.h>
#include <stdint.h>

#include "otf_engine_common.cuh"

namespace otf {

constexpr int32_t WIN_NONE = 0x3FFFFFFF;
constexpr int RANK_SORT_MAX = 64;  // windows up to this many server events: rank sort, else bitonic
constexpr int MAXK = 16;           // transcode workers
constexpr int RING = 1024;         // timer-wheel buckets (windows, ~20 s at 20 ms); farther timers wait on a far list
constexpr int MAXTAB = 64;         // catalog sequences / ladder ranks kept in shared memory (more
                                   // sequences: their tables stay in global memory)
constexpr int MAXN = 32766;        // clients (16-bit wheel links; 0x7FFE/0x7FFF are descriptor states)

// Descriptor word (16 bits, shared memory): bit 15 = cached; bits 0-14 = the
// in-flight state: DF_IDLE (no job), DF_NOWAIT (job, no waiter yet) or the
// client id at the TAIL of the job's waiter list.  Waiters form a circular
// list through bnext (tail.next = head), so the whole Future-callback list of
// an in-flight descriptor lives in shared memory (backend.py:123-133,209-216).
constexpr uint16_t DF_CACHED = 0x8000;
constexpr uint16_t DF_IDLE = 0x7FFF;
constexpr uint16_t DF_NOWAIT = 0x7FFE;
__device__ __forceinline__ bool df_inflight(uint16_t f) { return (f & 0x7FFF) != DF_IDLE; }
constexpr int16_t NIL = -1;
constexpr int WIN_MAX_WARPS = 2;   // warps per scenario: 1, or 2 for the big shared-memory classes
constexpr int PAR_MAX = 256;       // windows up to this many requests may take the parallel server pass (uint8 indices)
#ifndef WIN_SORT_UNROLL
#define WIN_SORT_UNROLL 2
#endif
constexpr int SORT_UNROLL = WIN_SORT_UNROLL;
#ifndef WIN_QSORT_UNROLL
#define WIN_QSORT_UNROLL 2                           // fast rank sort's loop unroll (A/B switch)
#endif
constexpr int QSORT_UNROLL = WIN_QSORT_UNROLL;
#ifdef WIN_NO_PHASE_CYCLES                           // per-phase cycle counters (tools/probe.py)
#define WCLOCK() 0LL
#else
#define WCLOCK() clock64()
#endif   // rank-sort inner loop unroll (A/B switch)

struct WWorker {
    double when, ctime;
    int64_t eps_pos;
    int64_t size;
    uint32_t seq;
    int32_t win, pc, desc, job, pad;
};

// Shared-memory header of one scenario (followed by the per-client and
// per-descriptor arrays, see win_smem_bytes).
struct WinHeader {
    otf_batch b;                     // copies: every lane reads these at L1 latency
    otf_scenario sc;
    EngineState st;
    int64_t stats[OTF_ST_NSLOTS];
    QoeAcc qa;
    WWorker wk[MAXK];
    int32_t gq[MAXK];
    int32_t fq_w[MAXK], fq_d[MAXK], fq_j[MAXK];
    int32_t gq_head, gq_n, fq_head, fq_n;
    int32_t jq_head, jq_n, jq_cap;
    int32_t sq_head, sq_n, tokens;       // demand-priority mode: speculative FIFO, wakeup tokens
    int32_t n_list, n_blist, n_ties;
#ifdef WIN_BULK_GATHER
    unsigned long long gbar;             // mbarrier of the window bucket's bulk copy (WIN_BULK_GATHER)
#endif
    uint32_t wseq;
    int32_t far_head, far_n, far_min, k_done;
    int32_t arr_next;                    // next client (arrival order) not yet on the wheel
    int32_t arr_win;                     // its window (WIN_NONE when every client is on the wheel)
    uint32_t lq_head, lq_tail, lq_stamp; // lazy-LRU touch queue (global ring of lq_cap entries)
    int32_t lq_cap;
    // small read-only tables
    int32_t t_segcount[MAXTAB];
    double t_seqdur[MAXTAB], t_segdur[MAXTAB], t_zipf[MAXTAB], t_rho[MAXTAB];
    int64_t t_bitrates[MAXTAB], t_manifest[MAXTAB];
    // timer wheel: server-event and client-local buckets per window
    uint32_t bits[RING / 32];
    uint32_t cnt_srv[RING / 2];          // entries filed in each window's bucket arrays:
    uint32_t cnt_loc[RING / 2];          //   16-bit counts, two windows per word
    int32_t ovf_head, ovf_n, ovf_min;    // pushes past a full bucket (linked through bnext)
    int32_t n_loc;                       // this window's client-local events (bucket array)
    int32_t list_cap;                    // capacity of the window's server-event list (dynamic region)
    int32_t ctl, cur_m;                  // window-loop control word + the window being run
    int32_t n_bsrv;                      // entries gathered from the window's server bucket
    uint8_t ev_flags[PAR_MAX];           // parallel server pass: per request outcome (EV_*)
    uint8_t ev_touch[PAR_MAX];           //   LRU touches before it (exclusive prefix)
    uint8_t par_list[PAR_MAX];           //   the list partitioned by owner lane (time order kept)
    uint32_t par_cnt[32];                //   per owner lane: count, then next slot
    int32_t hand_safe;                   // no transcode can end within the window it starts in
    uint32_t lc[16];                     // the server lane's event counters (LC_*): shared memory,
                                         //   not registers (they are rarely on a critical path)
    double wmin[WIN_MAX_WARPS];          // per-warp partial minima (hand_safe)
};

// server-lane counters in WinHeader::lc (folded into the stats at server_end)
enum { LC_HITS = 0, LC_MISS, LC_EVICT, LC_REJECT, LC_WASTED, LC_READY, LC_SPEC, LC_SKIP0, LC_POPS = LC_SKIP0 + 6 };

// Server events one window can hold: the list lives in the dynamic shared region.
__host__ __device__ inline int32_t win_list_cap(int32_t n_clients) {
    int32_t c = 64;
    while (c < n_clients / 16 && c < 4096) c <<= 1;
    return c;
}

struct LqEnt {
    int32_t desc;
    uint32_t stamp;
};

__host__ __device__ inline int64_t lq_capacity(int64_t n_desc) {   // power of two >= max(4D, 4096)
    int64_t c = 4096;
    while (c < 4 * n_desc) c <<= 1;
    return c;
}

// A server-bucket entry carries the request's sort key and descriptor words, so
// the window's gather is one coalesced read instead of bucket -> client state.
struct SrvEnt {
    double when;                                       // fire time (the request's arrival)
    double ctime;                                      // arm time (orders equal fire times, sim.py:304-309)
    int32_t pk;                                        // rank | index << 8 | seq << 16
    int16_t cid;
    uint16_t desc;                                     // descriptor id (< 65535)
};

// The windowed engine's per-client coroutine state: what every client event
// reads and writes, 64 B (four 16-byte vectors, half an L2 line).  The rest --
// the pick stream and registration time (session boundaries) and, in records
// mode, the request's id / response slot / request time -- is in WCold.  The
// server pass never writes here: responses reach the client as RespMsg.
// In registers (WClient) every field is a full word; in memory (WPacked) the
// small ones are packed, and the struct is unpacked / packed once per event.
struct WClient {
    double level, last_sync, stall_time;               // PlayerBuffer (client.py:74-121)
    double est;                                        // throughput EWMA; < 0: none yet (client.py:261-263)
    double next_when;                                  // the pending timer's fire time (for a request:
                                                       //   its arrival at the server)
    double session_start;                              // buffer reset time (startup delay)
    int32_t session;                                   // session id (registration counter)
    int32_t seq, index;                                // the session's sequence (< 2^16), next segment (< 2^16)
    int32_t pc, rank, attempt, flags;                  // < 2^8 each; flags: buffer phase (2 bits) | WF_*
    uint32_t stall_events;
};
struct WPacked {
    double level, last_sync, stall_time, est, next_when, session_start;
    int32_t session;
    uint32_t seq_index;                                // seq | index << 16
    uint32_t small;                                    // pc | rank << 8 | attempt << 16 | flags << 24
    uint32_t stall_events;
};
static_assert(sizeof(WPacked) == 64, "a client's hot state is half an L2 line");
enum { WF_PHASE = 3, WF_LIVE = 4, WF_OPEN = 8 };       // buffer playing-state, buffer live, session open

struct WCold {                                         // 128 B: session-boundary / records-mode state
    Pcg64 picks;                                       // orchestrator.py:338-342
    double reg_time;                                   // session registration time (metrics.py:88-92 order)
    double ctime;                                      // arm time of a request pushed past a full bucket
    int64_t req_id, req_slot;                          // records: MediaServer request id, response slot
    double requested;                                  // records: the segment's request time (seg_start)
    double pad[5];
};
static_assert(sizeof(WCold) == 128, "WCold is one L2 line");

// A client event handed to the client lanes: a server response (segment,
// waited transcode or OverloadError) at `when`, or a client-local timer
// (path < 0) whose time is in the client's state.
struct RespMsg {
    double when;
    int32_t cid, path;
};

struct WinGlobalLayout {
    int64_t clients, picks, blist, jobq, specq, lstamp, lq, bsrv, bloc, total;
};

// Per-window bucket arrays: server events up to the list capacity, client-local
// events up to twice that; a push past a full bucket goes to the overflow list.
__host__ __device__ inline int32_t win_list_cap(int32_t n_clients);
__host__ __device__ inline int32_t bucket_cap_srv(int32_t n_clients) { return win_list_cap(n_clients); }
__host__ __device__ inline int32_t bucket_cap_loc(int32_t n_clients) { return 2 * win_list_cap(n_clients); }

__host__ __device__ inline WinGlobalLayout win_global_layout(int32_t n_clients, int64_t n_desc) {
    WinGlobalLayout L;
    int64_t o = 0;
    L.clients = o; o += align256((int64_t)sizeof(WPacked) * n_clients);
    L.picks = o;   o += align256((int64_t)sizeof(WCold) * n_clients);
    L.blist = o;   o += align256((int64_t)sizeof(RespMsg) * (n_clients + 64));
    L.jobq = o;    o += align256((int64_t)sizeof(JobEnt) * (n_desc + 1));
    L.specq = o;   o += align256((int64_t)sizeof(JobEnt) * (n_desc + 1));
    L.lstamp = o;  o += align256((int64_t)sizeof(uint32_t) * n_desc);
    L.lq = o;      o += align256((int64_t)sizeof(LqEnt) * 2 * lq_capacity(n_desc));
    L.bsrv = o;    o += align256((int64_t)sizeof(SrvEnt) * RING * bucket_cap_srv(n_clients));
    L.bloc = o;    o += align256((int64_t)sizeof(int32_t) * RING * bucket_cap_loc(n_clients));
    L.total = o;
    return L;
}

// the scenario's server-event list capacity (otf_scenario.list_cap, default by client count)
__host__ __device__ inline int32_t win_list_cap_sc(const otf_scenario &sc) {
    return sc.list_cap > 0 ? sc.list_cap : win_list_cap(sc.n_clients);
}

__host__ __device__ inline int64_t win_smem_bytes(int32_t n_clients, int64_t n_desc, int32_t list_cap) {
    int64_t o = (sizeof(WinHeader) + 15) & ~(int64_t)15;
    o += 16 * (int64_t)list_cap;          // when f64, pack i32, id i16, desc u16
    o += 2 * (int64_t)n_clients;          // wheel / waiter next links (int16)
    o = (o + 15) & ~(int64_t)15;
    o += 2 * (n_desc + 1);                // descriptor words (DF_*), +1: the server lane reads d + 1 early
    return (o + 15) & ~(int64_t)15;
}

// The windowed engine's limits (anything outside them runs on the exact engine;
// the host checks the same predicate up front, otf_windowed_fits):
//   16-bit client ids (15-bit waiter links) and 16-bit descriptor ids, the server-event key packing
//   rank | index << 8 | seq << 16 (index < 256), the shared catalog tables, the
//   worker masks, and a positive request latency (the lookahead).
__host__ __device__ inline bool win_fits(const otf_scenario &sc) {
    const int64_t D = (int64_t)sc.n_seq * sc.n_ranks * sc.max_nseg;
    return sc.n_workers <= MAXK && sc.n_clients <= MAXN && sc.n_seq < 32768 && sc.n_ranks <= MAXTAB &&
           sc.max_nseg <= 256 && D < 65535 && sc.latency > 0 &&
           sc.horizon / (sc.latency * (1.0 - 0x1p-20)) < 5.0e8;
}

struct Win {
    Scn S;
    WinHeader *h;
    int16_t *bnext;
    double *lw;                                        // window's server events: time,
    int32_t *lp;                                       //   rank | index << 8 | seq << 16,
    int16_t *li;                                       //   client id
    uint16_t *ld;                                      //   descriptor id
    uint32_t *lstamp;                                  // latest touch stamp per descriptor (global)
    LqEnt *lq;                                         // touch queue (global, 2 * lq_cap)
    uint16_t *dflags;                                  // descriptor words (DF_*), shared
    WPacked *cl;                                       // hot client state (global)
    WCold *wc;                                         // cold client state (global)
    RespMsg *blist;                                    // this window's responses (+ overflowed local timers)
    SrvEnt *bsrv;                                      // bucket arrays [RING][cap]
    int32_t *bloc;
    int32_t scap, lcap;
    JobEnt *jq, *sq;
    double W, invW, H, E, now;
    double L, target;                                  // request latency, buffer target (registers)
    int32_t k;
    // lane 0's register copies of the hot server counters during phase A
    bool wdirty;                                       // `due` changed: recompute the earliest due worker
    uint32_t due;                                      // workers whose service timer fires in this window
    // server lane's register copies during phase A (loaded/stored around it)
    double svc_floor;                                  // min over ranks rho * min segment duration
};

// window index of a timer: the k with k*W <= when < (k+1)*W (both bounds as doubles);
// one out-of-line copy (scalar arguments) serves every call site
__device__ __noinline__ int32_t win_of(double when, double W, double invW) {
    double q = floor(when * invW);                     // estimate; the exact bounds decide
    int32_t k = q < 1.0e9 ? (int32_t)q : 1000000000;
    if (k < 0) k = 0;
    while (k > 0 && when < (double)k * W) k--;
    while (when >= (double)(k + 1) * W) k++;
    return k;
}

__device__ __forceinline__ int32_t timer_win(const Win &w, double when) {
    if (!(when <= w.H)) return WIN_NONE;     // run_until(H) never fires it (sim.py:352)
    int32_t k = win_of(when, w.W, w.invW);
    return k < WIN_NONE ? k : WIN_NONE;
}

// Put client c on the bucket of window `wk` (any lane; lock-free push).  A server
// event (request) carries its sort key, arm time and descriptor.
__device__ __forceinline__ void bucket_push(Win &w, int32_t c, int32_t wk, bool srv, const WClient &cl, double ctime,
                                            int32_t desc) {
    WinHeader *h = w.h;
    if (wk - w.k < RING) {
        int32_t slot = wk & (RING - 1);
        const int32_t cap = srv ? w.scap : w.lcap;
        const uint32_t sh = (slot & 1) << 4;
        int32_t pos = (int32_t)((atomicAdd(srv ? &h->cnt_srv[slot >> 1] : &h->cnt_loc[slot >> 1], 1u << sh) >> sh) & 0xffffu);
        if (pos < cap) {
            if (srv) {
                SrvEnt e;
                e.when = cl.next_when;
                e.ctime = ctime;
                e.pk = (int32_t)cl.rank | ((int32_t)cl.index << 8) | ((int32_t)cl.seq << 16);
                e.cid = (int16_t)c;
                e.desc = (uint16_t)desc;
                w.bsrv[(int64_t)slot * cap + pos] = e;
            } else {
                w.bloc[(int64_t)slot * cap + pos] = c;
            }
        } else {                                       // bucket full (rare): overflow list
            if (srv) w.wc[c].ctime = ctime;            //   (the entry is rebuilt from the client state)
            int32_t old = atomicExch(&h->ovf_head, c);
            w.bnext[c] = (int16_t)old;
            atomicAdd(&h->ovf_n, 1);
            atomicMin(&h->ovf_min, wk);
        }
        atomicOr(&h->bits[slot >> 5], 1u << (slot & 31));
    } else {                                           // beyond the wheel (rare): far list
#ifdef WIN_FAR_DIAG
        atomicAdd((unsigned long long *)&h->stats[28], wk >= WIN_NONE ? (1ull << 32) : 1ull);
#endif
        int32_t old = atomicExch(&h->far_head, c);
        w.bnext[c] = (int16_t)old;
        atomicAdd(&h->far_n, 1);
        atomicMin(&h->far_min, wk);
    }
}

// ---- server lane: cache / backend (lane 0 only) --------------------------------
// ---- SegmentCache as a lazy LRU (cache.py:27-92) ---------------------------------
// OrderedDict order == order of each key's latest touch (get moves to the end,
// put inserts at the end).  Every touch stamps the descriptor and appends
// (desc, stamp) to a queue; eviction pops the queue head and skips entries
// that are stale (not cached, or superseded by a later touch).  Hits are two
// stores -- no dependent loads on the server lane -- and evictions read the
// queue sequentially.  The queue is compacted (warp-parallel, order kept)
// before it can overflow.
__device__ __noinline__ uint32_t lq_compact_serial(LqEnt *lq, const uint16_t *dflags, const uint32_t *lstamp,
                                                   uint32_t head, uint32_t tail, uint32_t mask);

__device__ __forceinline__ void lru_touch(Win &w, int32_t d) {
    WinHeader *hh = w.h;
    const uint32_t mask = (uint32_t)hh->lq_cap - 1u;
    uint32_t s = ++hh->lq_stamp;
    w.lstamp[d] = s;
    if (hh->lq_tail - hh->lq_head > mask)
        hh->lq_tail = lq_compact_serial(w.lq, w.dflags, w.lstamp, hh->lq_head, hh->lq_tail, mask);
    LqEnt e; e.desc = d; e.stamp = s;
    w.lq[hh->lq_tail & mask] = e;
    hh->lq_tail++;
}
__device__ __forceinline__ bool cache_get(Win &w, int32_t d) {          // cache.py:45-52
    if (!(w.dflags[d] & DF_CACHED)) { w.h->lc[LC_MISS]++; return false; }
    lru_touch(w, d);
    w.h->lc[LC_HITS]++;
    return true;
}
__device__ void cache_put(Win &w, int32_t d, int64_t size) {             // cache.py:58-81
    const int64_t cap = w.S.sc->cache_capacity;
    if (size > cap) { w.h->lc[LC_REJECT]++; return; }
    if (w.dflags[d] & DF_CACHED) {                     // replace: its old queue entry goes stale
        w.h->st.cur_bytes -= size;
        w.dflags[d] &= (uint16_t)~DF_CACHED;
        w.h->st.entries--;
    }
    while (w.h->st.cur_bytes + size > cap) {                 // popitem(last=False): oldest live entry
        LqEnt e = w.lq[w.h->lq_head & ((uint32_t)w.h->lq_cap - 1u)];
        w.h->lq_head++;
        int32_t v = e.desc;
        if (!(w.dflags[v] & DF_CACHED) || w.lstamp[v] != e.stamp) continue;
        w.dflags[v] &= (uint16_t)~DF_CACHED;
        w.h->st.entries--;
        w.h->st.cur_bytes -= w.S.size(v);
        w.h->lc[LC_EVICT]++;
    }
    lru_touch(w, d);
    w.dflags[d] |= DF_CACHED;
    w.h->st.entries++;
    w.h->st.cur_bytes += size;
}

// Drop stale queue entries in place, keeping order (lane 0; only if a window
// overran the pre-window compaction margin).
__device__ __noinline__ uint32_t lq_compact_serial(LqEnt *lq, const uint16_t *dflags, const uint32_t *lstamp,
                                                   uint32_t head, uint32_t tail, uint32_t mask) {
    uint32_t o = head;
    for (uint32_t i = head; i != tail; i++) {
        LqEnt e = lq[i & mask];
        if ((dflags[e.desc] & DF_CACHED) && lstamp[e.desc] == e.stamp) lq[(o++) & mask] = e;
    }
    return o;
}

// Warp-parallel order-preserving compaction of the touch queue into a fresh
// region (called between windows when the queue is 3/4 full).
__device__ void lq_compact_warp(Win &w, int lane) {
    WinHeader *h = w.h;
    const uint32_t cap = (uint32_t)h->lq_cap;
    const uint32_t head = h->lq_head, tail = h->lq_tail;
    uint32_t out = 0;                                  // compacted entries go to [0, out) of the spare half
    LqEnt *dst = w.lq + cap;                           // the queue owns 2*cap slots: compact into the other half
    for (uint32_t base = head; base < tail; base += 32) {
        uint32_t i = base + lane;
        bool keep = false;
        LqEnt e;
        if (i < tail) {
            e = w.lq[i & (cap - 1)];
            keep = (w.dflags[e.desc] & DF_CACHED) && w.lstamp[e.desc] == e.stamp;
        }
        unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) dst[out + __popc(m & ((1u << lane) - 1))] = e;
        out += __popc(m);
    }
    __syncwarp();
    for (uint32_t i = lane; i < out; i += 32) w.lq[i] = dst[i];
    __syncwarp();
    if (lane == 0) { h->lq_head = 0; h->lq_tail = out; }
    __syncwarp();
}

// Backend._enqueue (backend.py:156-170); true on OverloadError (no idle worker,
// queue at its bound: Queue.put_nowait raises QueueFull, sim.py:229-240).
__device__ bool enqueue_job(Win &w, int32_t d, int32_t origin) {
    WinHeader *h = w.h;
    const bool prio = w.S.sc->demand_priority != 0;
    if (prio) {                                        // workers never wait on the job queues
        if (origin == OTF_ORIGIN_DEMAND && w.S.sc->queue_bound > 0 && h->jq_n >= w.S.sc->queue_bound) return true;
    } else if (h->gq_n == 0 && w.S.sc->queue_bound > 0 && h->jq_n >= w.S.sc->queue_bound) {
        return true;
    }
    int32_t j = w.S.record_job(d, origin, w.now);
    w.dflags[d] = (uint16_t)((w.dflags[d] & DF_CACHED) | DF_NOWAIT);   // in flight, no waiter yet
    if (prio) {                                        // separate FIFOs + _wakeup.put_nowait(None, force=True)
        JobEnt e; e.desc = d; e.job = j;
        if (origin == OTF_ORIGIN_SPECULATIVE) {
            int32_t pos = h->sq_head + h->sq_n; if (pos >= h->jq_cap) pos -= h->jq_cap;
            w.sq[pos] = e; h->sq_n++;
        } else {
            int32_t pos = h->jq_head + h->jq_n; if (pos >= h->jq_cap) pos -= h->jq_cap;
            w.jq[pos] = e; h->jq_n++;
        }
        if (h->gq_n > 0) {                             // wake the first idle worker (ready hop)
            int32_t wid = h->gq[h->gq_head];
            h->gq_head = (h->gq_head + 1 == w.S.sc->n_workers) ? 0 : h->gq_head + 1;
            h->gq_n--;
            int32_t pos = h->fq_head + h->fq_n;
            if (pos >= MAXK) pos -= MAXK;
            h->fq_w[pos] = wid; h->fq_d[pos] = -1; h->fq_j[pos] = -1;
            h->fq_n++;
        } else {
            h->tokens++;
        }
        return false;
    }
    if (h->gq_n > 0) {                                 // Queue.put_nowait -> first getter
        int32_t wid = h->gq[h->gq_head];
        h->gq_head = (h->gq_head + 1 == w.S.sc->n_workers) ? 0 : h->gq_head + 1;
        h->gq_n--;
        int32_t pos = h->fq_head + h->fq_n;
        if (pos >= MAXK) pos -= MAXK;
        h->fq_w[pos] = wid; h->fq_d[pos] = d; h->fq_j[pos] = j;
        h->fq_n++;
    } else {
        if (h->jq_n >= h->jq_cap) { w.S.flag(OTF_S_INTERNAL); return false; }
        int32_t pos = h->jq_head + h->jq_n;
        if (pos >= h->jq_cap) pos -= h->jq_cap;
        JobEnt e; e.desc = d; e.job = j;
        w.jq[pos] = e;
        h->jq_n++;
    }
    return false;
}

// Response of MediaServer.segment (server.py:76-77): fix the record's slot
// in response order and hand the client back to the client lanes at `now`
// (a RespMsg: the client's own state is written by its lane only).  The
// record itself and the request QoE are written by the client lane.
__device__ __forceinline__ void respond(Win &w, int32_t cid, int32_t path) {
    const int64_t slot = w.h->st.n_req++;
    if (w.S.records) w.wc[cid].req_slot = slot;
    RespMsg m;
    m.when = w.now;
    m.cid = cid;
    m.path = path;
    w.blist[w.h->n_blist++] = m;
}

// Waiter links reuse bnext (a waiting client has no pending timer): bits 0-14 are
// the next waiter, bit 15 marks a client whose request created the demand job
// (path "transcoded"; the others joined an in-flight job: "waited_inflight").
constexpr uint16_t WL_TRANSCODED = 0x8000;

__device__ void resolve(Win &w, int32_t d) {                             // backend.py:209-216
    const uint16_t f = w.dflags[d];
    if (!df_inflight(f)) return;
    w.dflags[d] = (uint16_t)((f & DF_CACHED) | DF_IDLE);
    const int32_t t = f & 0x7FFF;
    if (t == DF_NOWAIT) return;
    int32_t c = (uint16_t)w.bnext[t] & 0x7FFF;         // head: waiter Future callbacks, await order
    for (;;) {
        const uint16_t lk = (uint16_t)w.bnext[c];
        respond(w, c, (lk & WL_TRANSCODED) ? OTF_PATH_TRANSCODED : OTF_PATH_WAITED);
        if (c == t) break;
        c = lk & 0x7FFF;
    }
}

// Append a waiter.
__device__ __forceinline__ void add_waiter(Win &w, int32_t d, int32_t cid, bool transcoded) {
    const uint16_t f = w.dflags[d];
    const int32_t t = f & 0x7FFF;
    const uint16_t tag = transcoded ? WL_TRANSCODED : 0;
    if (t == DF_NOWAIT) {
        w.bnext[cid] = (int16_t)(cid | tag);
    } else {
        const uint16_t lt = (uint16_t)w.bnext[t];
        w.bnext[cid] = (int16_t)((lt & 0x7FFF) | tag);
        w.bnext[t] = (int16_t)((lt & WL_TRANSCODED) | cid);
    }
    w.dflags[d] = (uint16_t)((f & DF_CACHED) | cid);
}

// Backend._next_job (backend.py:174-184): a job now (no yield), or the worker
// becomes an idle getter (FIFO) and false is returned.
__device__ bool take_job(Win &w, int32_t wid, int32_t &d, int32_t &j) {
    WinHeader *h = w.h;
    const otf_scenario &sc = *w.S.sc;
    for (;;) {
        if (h->jq_n > 0) {                             // Queue.get on a non-empty queue: no yield
            JobEnt e = w.jq[h->jq_head];
            h->jq_head = (h->jq_head + 1 == h->jq_cap) ? 0 : h->jq_head + 1;
            h->jq_n--;
            d = e.desc; j = e.job;
            return true;
        }
        if (sc.demand_priority) {
            if (h->sq_n > 0) {                         // speculative jobs only when no demand waits
                JobEnt e = w.sq[h->sq_head];
                h->sq_head = (h->sq_head + 1 == h->jq_cap) ? 0 : h->sq_head + 1;
                h->sq_n--;
                d = e.desc; j = e.job;
                return true;
            }
            if (h->tokens > 0) { h->tokens--; continue; }   // stale wakeup token: no yield
        }
        int32_t pos = h->gq_head + h->gq_n;
        if (pos >= sc.n_workers) pos -= sc.n_workers;
        h->gq[pos] = wid;
        h->gq_n++;
        h->wk[wid].pc = W_GOT;
        h->wk[wid].win = WIN_NONE;
        if (w.due & (1u << wid)) { w.due &= ~(1u << wid); w.wdirty = true; }
        return false;
    }
}

// Backend._worker_loop body from "job dequeued" until the worker yields.
__device__ void worker_run(Win &w, int32_t wid, int32_t d, int32_t j) {
    WinHeader *h = w.h;
    const otf_scenario &sc = *w.S.sc;
    for (;;) {
        if (w.S.sc->cache_enabled && (w.dflags[d] & DF_CACHED)) {  // dedup on dequeue (backend.py:193-198)
            w.S.job_outcome(j, OTF_OUTCOME_DROPPED);
            w.h->lc[LC_WASTED]++;
            resolve(w, d);
        } else {                                             // run_transcode (transcode.py:123-128)
            WWorker &k = h->wk[wid];
            w.S.job_started(j, w.now);
            Worker tmp; tmp.eps_pos = k.eps_pos;
            double svc = w.S.service_time(tmp, wid, d);
            k.eps_pos = tmp.eps_pos;
            k.when = w.now + svc;
            k.ctime = w.now;
            k.seq = h->wseq++;
            k.win = timer_win(w, k.when);
            k.desc = d;
            k.job = j;
            k.size = w.S.size(d);
            k.pc = W_SERVICE;
            if (k.win == w.k) { w.due |= 1u << wid; w.wdirty = true; }   // fires in this window (rare)
            return;
        }
        if (!take_job(w, wid, d, j)) return;
    }
}

__device__ void drain_handoffs(Win &w) {            // ready-queue hops of handed-off jobs
    WinHeader *h = w.h;
    while (h->fq_n > 0) {
        int32_t wid = h->fq_w[h->fq_head], d = h->fq_d[h->fq_head], j = h->fq_j[h->fq_head];
        h->fq_head = (h->fq_head + 1 == MAXK) ? 0 : h->fq_head + 1;
        h->fq_n--;
        w.h->lc[LC_READY]++;
        if (j < 0 && !take_job(w, wid, d, j)) continue;   // priority mode: a wakeup, not a job
        worker_run(w, wid, d, j);
    }
}

// Backend.maybe_speculate (backend.py:135-154) for a request on d whose rank is
// not stored, with the next descriptor's word `fn` and the sequence's segment
// count already loaded.
__device__ __forceinline__ void speculate_next(Win &w, int32_t d, int32_t index, int32_t segc, uint16_t fn) {
    if (!w.S.sc->spec_enabled) { w.h->lc[LC_SKIP0 + 0]++; return; }
    if (index + 1 >= segc) { w.h->lc[LC_SKIP0 + 1]++; return; }
    if (w.S.sc->cache_enabled && (fn & DF_CACHED)) { w.h->lc[LC_SKIP0 + 3]++; return; }
    if (df_inflight(fn)) { w.h->lc[LC_SKIP0 + 4]++; return; }
    if (enqueue_job(w, d + 1, OTF_ORIGIN_SPECULATIVE)) { w.h->lc[LC_SKIP0 + 5]++; return; }
    w.h->lc[LC_SPEC]++;
}

// One client server event: MediaServer.segment + Backend.handle (server.py:61-78,
// backend.py:115-133), with every shared-memory word it branches on loaded up front
// (the descriptor's word f, the next descriptor's word fn, the sequence's
// segment count), so the server lane pays one shared-memory round trip per
// request instead of a chain of them.
__device__ __forceinline__ void server_request_fast(Win &w, int32_t cid, int32_t d, int32_t pk, uint16_t f,
                                                    uint16_t fn, int32_t segc) {
    const int32_t rank = pk & 0xff, index = (pk >> 8) & 0xff;
    const int64_t rid = w.h->st.req_counter++;
    if (w.S.records) w.wc[cid].req_id = rid;
    if ((w.S.sc->stored_mask >> rank) & 1u) {
        respond(w, cid, OTF_PATH_STORAGE);
        return;
    }
    if (w.S.sc->cache_enabled) {                       // SegmentCache.get (cache.py:45-52)
        if (f & DF_CACHED) {
            lru_touch(w, d);
            w.h->lc[LC_HITS]++;
            speculate_next(w, d, index, segc, fn);
            respond(w, cid, OTF_PATH_CACHE);
            return;
        }
        w.h->lc[LC_MISS]++;
    }
    if (df_inflight(f)) {
        speculate_next(w, d, index, segc, fn);
        add_waiter(w, d, cid, false);
    } else if (enqueue_job(w, d, OTF_ORIGIN_DEMAND)) {
        respond(w, cid, OTF_PATH_ERROR);               // OverloadError: error record (server.py:70-73)
    } else {
        speculate_next(w, d, index, segc, fn);
        add_waiter(w, d, cid, true);
    }
}

// worker service timer fired (transcode.py:129-131, backend.py:205-207)
__device__ void server_worker_done(Win &w, int32_t wid) {
    WWorker &k = w.h->wk[wid];
    int32_t d = k.desc, j = k.job;
    k.win = WIN_NONE;
    w.due &= ~(1u << wid);
    w.wdirty = true;
    w.S.job_finished(j, w.now);
    if (w.S.sc->cache_enabled) cache_put(w, d, k.size);
    resolve(w, d);
    int32_t nd, nj;                                    // next job
    if (take_job(w, wid, nd, nj)) worker_run(w, wid, nd, nj);
}

// The server lane's scalar state stays in lane 0's registers for the whole run
// (loaded once by server_begin, flushed by server_end); per window only the
// queue cursors shared with the compaction step are exchanged.
__device__ void server_begin(Win &w) {
    WinHeader *h = w.h;
    const otf_scenario &sc0 = *w.S.sc;
    w.h->lc[LC_HITS] = w.h->lc[LC_MISS] = w.h->lc[LC_EVICT] = w.h->lc[LC_REJECT] = w.h->lc[LC_WASTED] = w.h->lc[LC_READY] = w.h->lc[LC_SPEC] = 0;
    for (int q = 0; q < 6; q++) w.h->lc[LC_SKIP0 + q] = 0;
    w.h->lc[LC_POPS] = 0;
    double rho_min = INFINITY, dur_min = INFINITY;     // service-time floor (parallel pass guard)
    for (int32_t r = 0; r < sc0.n_ranks; r++) rho_min = fmin(rho_min, w.S.rho[r]);
    for (int32_t q = 0; q < sc0.n_seq; q++) {
        const int32_t last = w.S.segcounts[q] - 1;
        dur_min = fmin(dur_min, fmin(w.S.segdur[q], seg_duration(w.S.seqdur[q], w.S.segdur[q], last)));
    }
    w.svc_floor = rho_min * dur_min;
}

__device__ void server_end(Win &w) {
    WinHeader *h = w.h;
    h->stats[OTF_ST_TIMER_POPS] += w.h->lc[LC_POPS];
    h->stats[OTF_ST_HITS] += w.h->lc[LC_HITS];
    h->stats[OTF_ST_MISSES] += w.h->lc[LC_MISS];
    h->stats[OTF_ST_EVICTIONS] += w.h->lc[LC_EVICT];
    h->stats[OTF_ST_REJECTED] += w.h->lc[LC_REJECT];
    h->stats[OTF_ST_WASTED] += w.h->lc[LC_WASTED];
    h->stats[OTF_ST_READY_CALLBACKS] += w.h->lc[LC_READY];
    h->stats[OTF_ST_SPEC_ENQUEUED] += w.h->lc[LC_SPEC];
    for (int q = 0; q < 6; q++) h->stats[OTF_ST_SKIP_DISABLED + q] += w.h->lc[LC_SKIP0 + q];
}

// One request of the window's sorted list (the list entry was loaded one event ahead).
#define PHASE_A_REQUEST()                                                              \
    do {                                                                               \
        w.now = cw;                                                                    \
        const int32_t cid = ncid, d = nd, pk = npk;                                    \
        const uint16_t f = w.dflags[d], fn = w.dflags[d + 1];                          \
        const int32_t segc = segcount[pk >> 16];                                       \
        i++;                                                                           \
        if (i < n) { cw = w.lw[i]; ncid = w.li[i]; nd = w.ld[i]; npk = w.lp[i]; }      \
        server_request_fast(w, cid, d, pk, f, fn, segc);                               \
    } while (0)

// ---- parallel server pass for request-only windows -------------------------------
// When no worker timer falls in the window, no worker is idle (every enqueue
// joins the FIFO: Queue.put_nowait with no getter, sim.py:229-240), and the
// backend has neither a queue bound nor demand priority, the window's server
// events are requests only and the cache contents cannot change (puts and
// evictions happen only when a transcode completes, backend.py:205-207).  A
// request then touches (a) its (sequence, rank)'s descriptors -- cached /
// in-flight state, waiter lists, the speculative next segment -- and (b)
// global sequence numbers: request ids, response slots, LRU touch stamps, job
// ids and FIFO positions.  (a) is replayed per (sequence, rank) group, in
// time order, by the lane that owns the group; (b) are exclusive prefix sums
// over the window's time order.  The result is the serial order's, exactly.
enum { EV_PATH = 7, EV_IMM = 8, EV_TOUCH = 16, EV_ENQ_D = 32, EV_ENQ_S = 64 };

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane, uint32_t &total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
    return __reduce_add_sync(0xffffffffu, v);          // one REDUX (sm_80+), not five shuffles
}

__device__ __forceinline__ void phase_a_parallel(Win &w, int lane) {
    WinHeader *h = w.h;
    const otf_scenario &sc = *w.S.sc;
    const int32_t n = h->n_list;
    const uint32_t stored_mask = sc.stored_mask;
    const bool cache_on = sc.cache_enabled != 0, spec_on = sc.spec_enabled != 0;
    const int32_t n_ranks = sc.n_ranks;
#ifdef WIN_DIAG
    long long dga = clock64();
#endif
    // (a) per-group replay: lane (seq * n_ranks + rank) % 32 owns the group.  First a
    // stable partition of the list by owner lane (time order kept inside each lane's
    // run), so that every lane then walks ITS requests while the others walk theirs.
    h->par_cnt[lane] = 0;
    __syncwarp();
    for (int32_t base = 0; base < n; base += 32) {      // counts per owner
        const int32_t i = base + lane;
        const int32_t pk = i < n ? w.lp[i] : 0;
        const int32_t own = i < n ? ((((pk >> 16) * n_ranks) + (pk & 0xff)) & 31) : 32 + lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, own);
        if (i < n && (peers & ((1u << lane) - 1u)) == 0) h->par_cnt[own] += __popc(peers);
        __syncwarp();
    }
    const uint32_t my_cnt = h->par_cnt[lane];
    uint32_t n_all;
    const uint32_t my_off = warp_excl_scan(my_cnt, lane, n_all);
    __syncwarp();
    h->par_cnt[lane] = my_off;                          // now: the next free slot of each owner's run
    __syncwarp();
    for (int32_t base = 0; base < n; base += 32) {      // scatter, stable
        const int32_t i = base + lane;
        const int32_t pk = i < n ? w.lp[i] : 0;
        const int32_t own = i < n ? ((((pk >> 16) * n_ranks) + (pk & 0xff)) & 31) : 32 + lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, own);
        if (i < n) h->par_list[h->par_cnt[own] + __popc(peers & ((1u << lane) - 1u))] = (uint8_t)i;
        __syncwarp();
        if (i < n && (peers & ((1u << lane) - 1u)) == 0) h->par_cnt[own] += __popc(peers);
        __syncwarp();
    }
    uint32_t hits = 0, miss = 0, sk0 = 0, sk1 = 0, sk3 = 0, sk4 = 0, spec = 0;
    OTF_NOUNROLL
    for (uint32_t k = my_off; k < my_off + my_cnt; k++) {
        const int32_t i = h->par_list[k];
        const int32_t pk = w.lp[i];
        const int32_t rank = pk & 0xff, seq = pk >> 16;
        const int32_t d = w.ld[i], cid = w.li[i], index = (pk >> 8) & 0xff;
        uint32_t fl;
        if ((stored_mask >> rank) & 1u) {
            fl = EV_IMM | OTF_PATH_STORAGE;
        } else {
            const uint16_t f = w.dflags[d];
            if (cache_on && (f & DF_CACHED)) {
                hits++;
                fl = EV_IMM | EV_TOUCH | OTF_PATH_CACHE;
            } else {
                if (cache_on) miss++;
                if (df_inflight(f)) {
                    fl = OTF_PATH_WAITED;
                } else {                               // demand job: in flight, no waiter yet
                    w.dflags[d] = (uint16_t)((f & DF_CACHED) | DF_NOWAIT);
                    fl = EV_ENQ_D | OTF_PATH_TRANSCODED;
                }
            }
            {                                          // maybe_speculate (backend.py:135-154)
                if (!spec_on) sk0++;
                else if (index + 1 >= w.S.segcounts[seq]) sk1++;
                else {
                    const uint16_t fn = w.dflags[d + 1];
                    if (cache_on && (fn & DF_CACHED)) sk3++;
                    else if (df_inflight(fn)) sk4++;
                    else {
                        w.dflags[d + 1] = (uint16_t)((fn & DF_CACHED) | DF_NOWAIT);
                        fl |= EV_ENQ_S;
                        spec++;
                    }
                }
            }
            if (!(fl & EV_IMM)) add_waiter(w, d, cid, (fl & EV_PATH) == OTF_PATH_TRANSCODED);
        }
        h->ev_flags[i] = (uint8_t)fl;
    }
    __syncwarp();
#ifdef WIN_DIAG
    if (lane == 0) h->stats[28] += clock64() - dga;
    dga = clock64();
#endif
    // (b) sequence numbers in time order: exclusive prefix sums over the list
    // (lane l holds requests E*l .. E*l+E-1)
    const int32_t E = (n + 31) >> 5;                    // requests per lane (runtime: one copy of the code)
    uint32_t c_imm = 0, c_tch = 0, c_enq = 0, c_enq_d = 0;
#pragma unroll 1
    for (int32_t t = 0; t < E; t++) {
        const int32_t i = E * lane + t;
        const uint32_t f = i < n ? h->ev_flags[i] : 0u;
        c_imm += (f >> 3) & 1u;
        c_tch += (f >> 4) & 1u;
        c_enq += ((f >> 5) & 1u) + ((f >> 6) & 1u);
        c_enq_d += (f >> 5) & 1u;
    }
    // one scan for all three counts: 10-bit fields (n <= PAR_MAX = 256 requests, so
    // every prefix and total is < 2 * 256 + 1 < 1024 and no field carries into the next)
    static_assert(2 * PAR_MAX < 1024, "packed scan fields");
    uint32_t n_pk;
    const uint32_t p_pk = warp_excl_scan(c_imm | (c_tch << 10) | (c_enq << 20), lane, n_pk);
    uint32_t p_imm = p_pk & 1023u, p_tch = (p_pk >> 10) & 1023u, p_enq = p_pk >> 20;
    const uint32_t n_imm = n_pk & 1023u, n_tch = (n_pk >> 10) & 1023u, n_enq = n_pk >> 20;
    const uint32_t n_enq_d = warp_sum(c_enq_d);
    // the server lane's scalars (lane 0's registers) as the bases
    const int64_t req_base = h->st.req_counter;        // (shared: every lane reads the same word)
    const int64_t slot_base = h->st.n_req;
    const int32_t blist_base = h->n_blist;             // the header copies (every lane reads them)
    const uint32_t lq_tail = h->lq_tail;
    const uint32_t stamp_base = h->lq_stamp;
    const uint32_t lq_mask = (uint32_t)h->lq_cap - 1u;
    const int32_t jq_base = h->jq_head + h->jq_n;
    const int64_t job_base = h->st.n_job;
    // the first n_hand enqueues (time order) go to the idle workers (getters, FIFO);
    // the rest join the job FIFO
    const uint32_t n_hand = min(n_enq, (uint32_t)h->gq_n);
#pragma unroll 1
    for (int32_t t = 0; t < E; t++) {
        const int32_t i = E * lane + t;
        if (i >= n) break;
        const uint32_t f = h->ev_flags[i];
        h->ev_touch[i] = (uint8_t)p_tch;
        const int32_t cid = w.li[i], d = w.ld[i];
        const double now = w.lw[i];
        if (w.S.records) {
            w.wc[cid].req_id = req_base + i;
            if (f & EV_IMM) w.wc[cid].req_slot = slot_base + p_imm;
        }
        if (f & EV_IMM) {                              // respond (server.py:76-77)
            RespMsg m;
            m.when = now;
            m.cid = cid;
            m.path = (int32_t)(f & EV_PATH);
            w.blist[blist_base + (int32_t)p_imm] = m;
        }
        if (f & EV_TOUCH) {                            // lru_touch, in time order
            LqEnt e; e.desc = d; e.stamp = stamp_base + p_tch + 1u;
            w.lq[(lq_tail + p_tch) & lq_mask] = e;
        }
        uint32_t q = p_enq;
        for (int k = 0; k < 2; k++) {                  // Backend._enqueue: demand job first, then the speculative one
            const uint32_t bit = k ? EV_ENQ_S : EV_ENQ_D;
            if (!(f & bit)) continue;
            const int32_t jd = k ? d + 1 : d;
            const int64_t j = job_base + q;
            if (q >= n_hand) {                         // Queue.put_nowait with no getter: the FIFO
                int32_t pos = jq_base + (int32_t)(q - n_hand);
                if (pos >= h->jq_cap) pos -= h->jq_cap;
                JobEnt je; je.desc = jd; je.job = (int32_t)j;
                w.jq[pos] = je;
            }
            if (w.S.records) {
                if (j < sc.job_cap) {
                    const int64_t o = sc.job_off + j;
                    w.S.b->job_seq[o] = w.S.desc_seq(jd);
                    w.S.b->job_rep[o] = w.S.desc_rank(jd);
                    w.S.b->job_index[o] = w.S.desc_index(jd);
                    w.S.b->job_origin[o] = k ? OTF_ORIGIN_SPECULATIVE : OTF_ORIGIN_DEMAND;
                    w.S.b->job_outcome[o] = OTF_OUTCOME_PENDING;
                    w.S.b->job_enq[o] = now;
                    w.S.b->job_start[o] = NAN;
                    w.S.b->job_fin[o] = NAN;
                } else {
                    w.S.flag(OTF_S_RECORD_OVERFLOW);
                }
            }
            q++;
        }
        p_imm += (f >> 3) & 1u;
        p_tch += (f >> 4) & 1u;
        p_enq += ((f >> 5) & 1u) + ((f >> 6) & 1u);
    }
    __syncwarp();
    // the latest touch stamp per descriptor: 32 requests at a time in time order; within
    // a chunk only the last toucher of a descriptor (highest lane of its match group)
    // stores, and a later chunk's stores follow the earlier one's
#ifndef WIN_SERIAL_STAMPS
    for (int32_t base = 0; base < n; base += 32) {
        const int32_t i = base + lane;
        const bool touch = i < n && (h->ev_flags[i] & EV_TOUCH);
        const int32_t d = touch ? (int32_t)w.ld[i] : -1 - lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (touch && (peers >> lane) == 1u) w.lstamp[d] = stamp_base + h->ev_touch[i] + 1u;
        __syncwarp();
    }
#else
    OTF_NOUNROLL
    for (uint32_t k = my_off; k < my_off + my_cnt; k++) {   // each lane over its own requests
        const int32_t i = h->par_list[k];
        if (h->ev_flags[i] & EV_TOUCH) w.lstamp[w.ld[i]] = stamp_base + h->ev_touch[i] + 1u;
    }
#endif
    // counters back into lane 0's registers / the header
    hits = warp_sum(hits); miss = warp_sum(miss); spec = warp_sum(spec);
    sk0 = warp_sum(sk0); sk1 = warp_sum(sk1); sk3 = warp_sum(sk3); sk4 = warp_sum(sk4);
    if (lane == 0) {
        h->st.req_counter += n;
        h->st.n_req += n_imm;
        h->n_blist += (int32_t)n_imm;
        h->lq_tail += n_tch;
        h->lq_stamp += n_tch;
        w.h->lc[LC_HITS] += hits; w.h->lc[LC_MISS] += miss; w.h->lc[LC_SPEC] += spec;
        w.h->lc[LC_SKIP0 + 0] += sk0; w.h->lc[LC_SKIP0 + 1] += sk1; w.h->lc[LC_SKIP0 + 3] += sk3; w.h->lc[LC_SKIP0 + 4] += sk4;
        w.h->lc[LC_POPS] += n;
        h->st.n_job += n_enq;
        h->jq_n += (int32_t)(n_enq - n_hand);
        // hand-offs, in time order: put_nowait -> the first getter's ready hop ->
        // worker_run (backend.py:186-204); parallel_ok made sure none ends in this window
        uint32_t q = 0;
        for (int32_t i = 0; i < n && q < n_hand; i++) {
            const uint32_t f = h->ev_flags[i];
            for (int k = 0; k < 2 && q < n_hand; k++) {
                if (!(f & (k ? EV_ENQ_S : EV_ENQ_D))) continue;
                const int32_t wid = h->gq[h->gq_head];
                h->gq_head = (h->gq_head + 1 == sc.n_workers) ? 0 : h->gq_head + 1;
                h->gq_n--;
                w.h->lc[LC_READY]++;
                w.now = w.lw[i];
                worker_run(w, wid, w.ld[i] + k, (int32_t)(job_base + q));
                q++;
            }
        }
        h->stats[OTF_ST_JOBS_TOTAL] += n_enq;
        h->stats[OTF_ST_JOBS_DEMAND] += n_enq_d;
        h->stats[OTF_ST_JOBS_SPEC] += n_enq - n_enq_d;
#ifdef WIN_DIAG
        h->stats[31] += clock64() - dga;
#endif
    }
    __syncwarp();
}

// Can this window take the parallel server pass?  (lane 0; see phase_a_parallel)
__device__ __forceinline__ bool parallel_ok(Win &w) {
    const WinHeader *h = w.h;
    const otf_scenario &sc = *w.S.sc;
    const int32_t n = h->n_list;
#ifdef WIN_DIAG
    {
        WinHeader *hm = w.h;
        if (h->gq_n > 0) hm->stats[30]++;
        if (n > PAR_MAX) hm->stats[31]++;
        for (int32_t q = 0; q < sc.n_workers; q++)
            if (h->wk[q].win == w.k) { hm->stats[24]++; break; }   // (diag build: overrides the sort cycles)
    }
#endif
    // every word loaded up front and combined without early exits: one shared-memory
    // round trip on the lane instead of a chain of them
    const int32_t n_ties = h->n_ties, fq_n = h->fq_n, gq_n = h->gq_n, hand_safe = h->hand_safe;
    const uint32_t lq_head = h->lq_head, lq_tail = h->lq_tail;
    const int32_t n_blist = h->n_blist;
#ifndef WIN_SERIAL_PAR_OK
    // the whole warp calls it: lane q checks worker q (K <= MAXK <= 32)
    const int lane = threadIdx.x & 31;
    const bool due = __any_sync(0xffffffffu, lane < sc.n_workers && h->wk[lane].win == w.k);
#else
    bool due = false;                                  // a transcode completes in this window
#pragma unroll 4
    for (int32_t q = 0; q < sc.n_workers; q++) due |= h->wk[q].win == w.k;
#endif
    // an idle worker handed a job here must not finish inside the window (hand_safe:
    // svc >= svc_floor * (1 + min eps) >= 2 W for every job, checked at kernel start)
    return (n >= 2) & (n <= PAR_MAX) & (n_ties == 0) & (fq_n == 0) & (sc.demand_priority == 0) &
           (sc.queue_bound <= 0) & !due & ((gq_n == 0) | (hand_safe != 0)) &
           (lq_tail - lq_head + (uint32_t)n <= (uint32_t)h->lq_cap - 1u);   // room for every touch
}

#ifndef WIN_NO_PREFIX
// A window where a transcode completes (1-2% of config-5 windows) is otherwise
// serial.  Its requests strictly before the earliest completion cannot see it, so
// when every other condition of the parallel pass holds, that prefix of the
// sorted list takes the parallel pass and the serial lane starts after it.
// Returns the prefix length (0: no split).  Lane 0.
__device__ __forceinline__ int32_t parallel_prefix(Win &w) {
    const WinHeader *h = w.h;
    const otf_scenario &sc = *w.S.sc;
    const int32_t n = h->n_list;
    if (n < 2 || h->n_ties != 0 || h->fq_n != 0 || sc.demand_priority != 0 || sc.queue_bound > 0 ||
        (h->gq_n != 0 && h->hand_safe == 0))
        return 0;
    double t_w = INFINITY;                             // the earliest completion due in this window
    for (int32_t q = 0; q < sc.n_workers; q++)
        if (h->wk[q].win == w.k) t_w = fmin(t_w, h->wk[q].when);
    int32_t lo = 0, hi = n < PAR_MAX ? n : PAR_MAX;   // requests with time < t_w: a prefix of the list
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (w.lw[mid] < t_w) lo = mid + 1; else hi = mid;
    }
    if (lo < 2 || h->lq_tail - h->lq_head + (uint32_t)lo > (uint32_t)h->lq_cap - 1u) return 0;
    return lo;
}
#endif

// Arm time of window request `cid` (rare tie-breaks only): the window's bucket
// entries carry it; a request pushed past a full bucket kept it in its WCold.
__device__ __noinline__ double req_ctime_at(const SrvEnt *as, int32_t ns, const WCold *wc, int32_t cid) {
    for (int32_t i = 0; i < ns; i++)
        if (as[i].cid == cid) return as[i].ctime;
    return wc[cid].ctime;
}
__device__ __forceinline__ double req_ctime(const Win &w, int32_t cid) {
    return req_ctime_at(w.bsrv + (int64_t)(w.k & (RING - 1)) * w.scap, w.h->n_bsrv, w.wc, cid);
}

// Phase A: replay the window's server events in (time, creation, tick) order.
__device__ void phase_a(Win &w, int32_t i0) {
    WinHeader *h = w.h;
    const int32_t K = w.S.sc->n_workers;
    const int32_t n = h->n_list;
    uint32_t due = 0;
    for (int32_t q = 0; q < K; q++) due |= (h->wk[q].win == w.k ? 1u : 0u) << q;
    w.due = due;
    w.wdirty = due != 0;
    int32_t bw = -1;
    double bw_when = 0.0, bw_ctime = 0.0;
    int32_t i = i0;                                    // requests before i0 took the parallel pass
    double cw = 0.0;                                   // next request, loaded one event ahead
    int32_t ncid = 0, nd = 0, npk = 0;
    if (i < n) { cw = w.lw[i]; ncid = w.li[i]; nd = w.ld[i]; npk = w.lp[i]; }
    const int32_t *segcount = w.S.segcounts;
    w.h->lc[LC_POPS] += n - i0;                                  // every request is one timer pop
    for (;;) {
        if (w.wdirty) {                                // earliest worker timer in this window
            bw = -1;
            for (uint32_t mm = w.due; mm; mm &= mm - 1) {
                const int32_t q = __ffs(mm) - 1;
                const WWorker &x = h->wk[q];
                if (bw < 0 || x.when < bw_when || (x.when == bw_when && (x.ctime < bw_ctime ||
                                                       (x.ctime == bw_ctime && x.seq < h->wk[bw].seq)))) {
                    bw = q; bw_when = x.when; bw_ctime = x.ctime;
                }
            }
            w.wdirty = false;
        }
        if (bw < 0) {                                  // no worker timer due: requests only (common)
            while (i < n) {
                PHASE_A_REQUEST();
                if (w.h->fq_n > 0) drain_handoffs(w);
                if (w.wdirty) break;                   // a started job ends inside this window (rare)
            }
            if (!w.wdirty) break;
            continue;
        }
        bool take_worker;
        if (i >= n) take_worker = true;
        else if (bw_when < cw) take_worker = true;
        else if (cw < bw_when) take_worker = false;
        else {
            double cc = req_ctime(w, w.li[i]);
            if (bw_ctime < cc) take_worker = true;
            else if (cc < bw_ctime) take_worker = false;
            else { w.S.flag(OTF_S_TIE); take_worker = true; }
        }
        if (take_worker) {
            w.h->lc[LC_POPS]++;
            w.now = bw_when;
            server_worker_done(w, bw);
        } else {
            PHASE_A_REQUEST();
        }
        if (w.h->fq_n > 0) drain_handoffs(w);
    }
}

// ---- client lanes ------------------------------------------------------------------
// The client coroutine (orchestrator.py:336-348, client.py:229-305) over the
// 64-byte WClient.  The buffer model functions (otf_model.cuh, pinned by the
// reference's known answers) run on a Buffer view of its fields.
__device__ __forceinline__ Buffer wbuf_get(const WClient &c) {
    Buffer b;
    b.level = c.level; b.last_sync = c.last_sync; b.stall_time = c.stall_time;
    b.started_at = NAN; b.session_start = c.session_start;
    b.phase = c.flags & WF_PHASE; b.stall_events = (int32_t)c.stall_events;
    return b;
}
__device__ __forceinline__ void wbuf_put(WClient &c, const Buffer &b) {
    c.level = b.level; c.last_sync = b.last_sync; c.stall_time = b.stall_time;
    c.flags = (c.flags & ~WF_PHASE) | (b.phase & WF_PHASE); c.stall_events = (uint32_t)b.stall_events;
}
__device__ __forceinline__ void wbuf_advance(WClient &c, double now) {
    Buffer b = wbuf_get(c);
    buf_advance(b, now);
    wbuf_put(c, b);
}
__device__ __forceinline__ int32_t wdesc(const Scn &S, const WClient &c) { return S.desc_id(c.seq, c.rank, c.index); }

// Arm a sleep for client c at `now` (loop.sleep, sim.py:317-324): returns true
// if the client keeps running inside this window (the timer fires before the
// window ends), else files the timer on the wheel and returns false.
__device__ __forceinline__ bool arm(Win &w, WClient &c, int32_t cid, double &now, double delay, int32_t next_pc) {
    c.pc = next_pc;
    if (delay <= 0) return true;                       // resolved future: no yield (sim.py:320-321)
    if (isinf(delay)) { c.pc = C_HUNG; return false; } // never resolves (sim.py:322)
    double when = now + delay;
    c.next_when = when;
    const bool srv = next_pc == C_SEG_LAT;             // a server event: always a later window
    // A client-local timer (anything but the request-latency timer, which reaches the
    // server) is run right away, even if it fires in a later window: nothing but the
    // client itself can act on a client in a local sleep (it neither waits on the
    // backend nor has a request pending), and nothing it does before its next request
    // is seen by anyone else ("Local chains").  The only cut is the
    // horizon: a timer after it never fires (sim.py:352).
    // ... except the session-end / next-session steps (playout, manifest latency and
    // transfer): those chains are twice as long as a segment's, and one of them in a
    // round of 32 lanes made the whole warp wait; they keep their own window's timer
    // (measured: 0.93 s -> 0.86 s on config 5).  The segment transfer is never
    // deferred: its start time and byte count live only in the chain's registers.
    // (late round 2: deferring only the playout -- the manifest steps now run in their
    // chain -- measured config 5 -1.6%, c5t -1.3%, config 4 -0.7%; deferring nothing
    // +16%: profiles/r02r_abn_defer*)
#ifndef WIN_DEFER_MASK
#define WIN_DEFER_MASK (1u << C_PLAYOUT)
#endif
    static_assert(!((WIN_DEFER_MASK >> C_SEG_XFER) & 1u), "the segment transfer completes in its chain");
    if (!srv && when <= w.H && (!((WIN_DEFER_MASK >> next_pc) & 1u) || when < w.E)) {
        now = when;
        return true;
    }
    const int32_t k = timer_win(w, when);
    if (k == WIN_NONE) return false;
    if (srv && k <= w.k) w.S.flag(OTF_S_TIE);          // lookahead violated (cannot happen)
    bucket_push(w, cid, k, srv, c, now, srv ? wdesc(w.S, c) : 0);   // the single push site (code size)
    return false;
}

// Client state moves through L2 with the evict-first policy: a client's next
// event is ~15 windows away, far beyond the L2's reach at full occupancy, so
// keeping its lines only evicts what does get reused (trace samples of the
// clients now transferring, segment sizes, bucket arrays).
__device__ __forceinline__ WClient wunpack(const WPacked &p) {
    WClient c;
    c.level = p.level; c.last_sync = p.last_sync; c.stall_time = p.stall_time; c.est = p.est;
    c.next_when = p.next_when; c.session_start = p.session_start; c.session = p.session;
    c.seq = (int32_t)(p.seq_index & 0xffffu); c.index = (int32_t)(p.seq_index >> 16);
    c.pc = (int32_t)(p.small & 0xffu); c.rank = (int32_t)((p.small >> 8) & 0xffu);
    c.attempt = (int32_t)((p.small >> 16) & 0xffu); c.flags = (int32_t)(p.small >> 24);
    c.stall_events = p.stall_events;
    return c;
}
__device__ __forceinline__ WPacked wpack(const WClient &c) {
    WPacked p;
    p.level = c.level; p.last_sync = c.last_sync; p.stall_time = c.stall_time; p.est = c.est;
    p.next_when = c.next_when; p.session_start = c.session_start; p.session = c.session;
    p.seq_index = (uint32_t)c.seq | ((uint32_t)c.index << 16);
    p.small = (uint32_t)c.pc | ((uint32_t)c.rank << 8) | ((uint32_t)c.attempt << 16) | ((uint32_t)c.flags << 24);
    p.stall_events = c.stall_events;
    return p;
}
static_assert(sizeof(WPacked) % 16 == 0, "WPacked moves as 16-byte vectors");
__device__ __forceinline__ void load_client_stream(WClient &dst, const WPacked *src) {
    WPacked t;
    int4 *d = reinterpret_cast<int4 *>(&t);
    const int4 *p = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(WPacked) / 16); q++) d[q] = __ldcs(p + q);
    dst = wunpack(t);
}
__device__ __forceinline__ void store_client_stream(WPacked *dst, const WClient &src) {
    const WPacked t = wpack(src);
    int4 *p = reinterpret_cast<int4 *>(dst);
    const int4 *s = reinterpret_cast<const int4 *>(&t);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(WPacked) / 16); q++) __stcs(p + q, s[q]);
}

// The response's record + QoE (server.py:76-77, metrics.py:67-78), written by the
// client lane in parallel; the request id and response slot (records) were fixed by
// the server lane.  The client's pending fire time is the request's arrival.
__device__ __forceinline__ void record_response(Win &w, const WClient &c, int32_t cid, double now, int32_t path) {
    Scn &S = w.S;
    const otf_scenario &sc = *S.sc;
    if (S.records) {
        const WCold &k = w.wc[cid];
        int64_t r = k.req_slot;
        if (r < sc.req_cap) {
            int64_t o = sc.req_off + r;
            S.b->req_id[o] = k.req_id;
            S.b->req_seq[o] = c.seq;
            S.b->req_rep[o] = c.rank;
            S.b->req_index[o] = c.index;
            S.b->req_path[o] = path;
            S.b->req_arrival[o] = c.next_when;
            S.b->req_response[o] = now;
            S.b->req_bytes[o] = path == OTF_PATH_ERROR ? 0 : S.size(wdesc(S, c));
        } else {
            S.flag(OTF_S_RECORD_OVERFLOW);
        }
    }
    double lat = now - c.next_when;
    QoeAcc &q = w.h->qa;
    atomicAdd(&q.lat_hist[lat_bin(lat)], 1u);
    atomicAdd(&q.path_count[path], 1u);
#ifndef WIN_NO_LAT_TAIL                                // A/B switch (timing only: breaks the summary)
    if (lat != 0.0) S.tail_latency(lat);
#endif
}

// _sync_report (client.py:284-288), records mode
__device__ __forceinline__ void wsync_session(Win &w, const WClient &c, double now) {
    const otf_scenario &sc = *w.S.sc;
    if (!w.S.records || c.session >= sc.sess_cap) return;
    const int64_t o = sc.sess_off + c.session;
    w.S.b->sess_end[o] = now;
    w.S.b->sess_stalls[o] = (int32_t)c.stall_events;
    w.S.b->sess_stall_time[o] = c.stall_time;
}

// the session's numbers are final (finished, aborted or harvested): its record
__device__ __forceinline__ void wqoe_session(Win &w, const WClient &c, int32_t cid, bool finished) {
    const bool live = (c.flags & WF_LIVE) != 0;
    w.S.tail_session(w.wc[cid].reg_time, live ? c.stall_time : 0.0, c.session, live ? c.stall_events : 0u,
                     finished);
}

// orchestrator.py:341-345 + client.py:237-239: pick a sequence, register a report.
// Out of line with plain arguments; returns sid << 16 | seq.
static __device__ __noinline__ int64_t wnew_session(WCold *k, const double *zipf, EngineState *st,
                                                    const otf_scenario *sc, const otf_batch *b, bool records,
                                                    int32_t cid, double now) {
    const int32_t seq = draw_sequence(&k->picks, sc->n_seq, sc->popularity, zipf);
    k->reg_time = now;
    const int64_t sid = atomicAdd((unsigned long long *)&st->n_sess, 1ull);
    if (records) {
        if (sid < sc->sess_cap) {
            const int64_t o = sc->sess_off + sid;
            b->sess_client[o] = cid;
            b->sess_seq[o] = seq;
            b->sess_start[o] = now;
            b->sess_end[o] = 0.0;
            b->sess_stalls[o] = 0;
            b->sess_stall_time[o] = 0.0;
            b->sess_startup[o] = NAN;
            b->sess_flags[o] = 0;
        } else {
            atomicOr(&st->status, OTF_S_RECORD_OVERFLOW);
        }
    }
    return sid << 16 | seq;
}


// client.py:261-268 for a transfer of `size` bytes started at `xfer_start`; returns
// true when the session has more segments, else leaves the buffer advanced for the
// final sleep(level) (client.py:270-271)
__device__ __forceinline__ bool wsegment_done(Win &w, WClient &c, int32_t cid, double now, double xfer_start,
                                              int64_t size) {
    Scn &S = w.S;
    double dt = now - xfer_start;                      // SegmentFetch.rate_bps
    double rate = dt > 0 ? ((double)size * 8.0) / dt : INFINITY;
    const double alpha = S.sc->alpha;                  // shared memory: not held in a register
    c.est = c.est < 0 ? rate : alpha * rate + (1.0 - alpha) * c.est;
    const double duration = seg_duration(S.seqdur[c.seq], S.segdur[c.seq], c.index);
    Buffer b = wbuf_get(c);
    const int32_t ph0 = b.phase;
    buf_on_segment(b, now, duration, S.sc->startup, S.sc->resume);
    wbuf_put(c, b);
    if (ph0 == PH_STARTUP && b.phase == PH_PLAYING) {  // playback started (client.py:117-119): the
        const double startup = b.started_at - b.session_start;   // startup delay is final now
        S.tail_startup(startup);
        if (S.records && c.session < S.sc->sess_cap) S.b->sess_startup[S.sc->sess_off + c.session] = startup;
    }
    const int64_t g = atomicAdd((unsigned long long *)&S.st->n_seg, 1ull);
    if (S.records) {
        if (g < S.sc->seg_cap) {
            const int64_t o = S.sc->seg_off + g;
            S.b->seg_session[o] = c.session;
            S.b->seg_index[o] = c.index;
            S.b->seg_rep[o] = c.rank;
            S.b->seg_start[o] = w.wc[cid].requested;
            S.b->seg_end[o] = now;
        } else {
            S.flag(OTF_S_RECORD_OVERFLOW);
        }
    }
    if (c.rank >= OTF_RANK_BINS) atomicOr(&S.qa->flags, (uint32_t)OTF_Q_RANKS_CAPPED);
    atomicAdd(&S.qa->rank_count[c.rank < OTF_RANK_BINS ? c.rank : OTF_RANK_BINS - 1], 1u);
    atomicAdd(&S.qa->n_segments, 1u);
    wsync_session(w, c, now);
    c.index++;
    // the final advance(now) (client.py:270) is a no-op here: on_segment just synced
    // the buffer at this same instant (dt = 0 changes neither level nor stall time)
    if (c.index < S.segcount(c.seq)) return true;
    return false;
}

// The client coroutine between two yields, entered at `now` with a response
// (path >= 0: record it, then the transfer or the retry logic) or at a local
// timer (path < 0).  Every state computes either "continue at the next state
// now" or (delay, next state); the single arm() site and the single shaped-
// transfer site keep the hot code small.
__device__ __forceinline__ void client_local_body(Win &w, WClient &c, int32_t cid, double now, int32_t path) {
    Scn &S = w.S;
    const otf_scenario &sc = *S.sc;
    double xfer_start = 0.0;                           // the segment transfer in flight (this chain)
    int64_t size = 0;
    if (path >= 0) {                                   // a response (segment or OverloadError): one inlined copy
        record_response(w, c, cid, now, path);
        c.pc = path == OTF_PATH_ERROR ? C_SEG_ERR : C_SEG_RESP;
    }
    for (;;) {
        double delay = 0.0;
        int32_t next = C_DONE;
        bool xfer = false;
        switch (c.pc) {
        case C_ARRIVED:                                // pick stream already seeded at init
            c.pc = C_SESSION;
            continue;
        case C_SESSION: {
            if (!(now < w.H)) { c.pc = C_DONE; return; }
            const int64_t r = wnew_session(w.wc + cid, S.zipf, S.st, S.sc, S.b, S.records, cid, now);
            c.session = (int32_t)(r >> 16);
            c.seq = (int32_t)(r & 0xffff);
            c.flags = (c.flags & ~WF_LIVE) | WF_OPEN;
            delay = w.L;                               // manifest request latency (netem.py:138-139)
            next = C_MAN_LAT;
            break;
        }
        case C_MAN_LAT:
            next = C_MAN_XFER;
            xfer = true;
            break;
        case C_MAN_XFER:                               // client.py:245-248
            c.level = 0.0; c.last_sync = now; c.stall_time = 0.0; c.session_start = now;
            c.stall_events = 0;
            c.flags = (c.flags & ~WF_PHASE) | PH_STARTUP | WF_LIVE;
            c.est = -1.0;
            c.rank = 1;
            c.index = 0;
            c.pc = C_INDEX_HEAD;
            continue;
        case C_INDEX_HEAD:
        case C_TARGET_WAIT:
            wbuf_advance(c, now);
            if ((c.flags & WF_PHASE) == PH_PLAYING && c.level >= w.target) {
                delay = c.level - w.target + 1e-9;
                next = C_TARGET_WAIT;
                break;
            }
            if (c.index > 0)                           // client.py:255-256
                c.rank = select_quality(c.level, c.rank, c.est >= 0, c.est, S.bitrates, sc.n_ranks,
                                                 S.sc->panic, S.sc->safe, S.sc->headroom);
            c.attempt = 0;                             // _fetch_with_retry (client.py:291-305)
            if (S.records) w.wc[cid].requested = now;
            delay = w.L;                               // request latency, then MediaServer.segment
            next = C_SEG_LAT;
            break;
        case C_SEG_RESP:
            xfer_start = now;
            next = C_SEG_XFER;
            xfer = true;
            break;
        case C_SEG_XFER:
            if (wsegment_done(w, c, cid, now, xfer_start, size)) { c.pc = C_INDEX_HEAD; continue; }
            delay = c.level;                           // play out the buffer (client.py:271)
            next = C_PLAYOUT;
            break;
        case C_PLAYOUT:                                // client.py:272-280 (+ the finally clause)
            {                                          // the next session's pick stream (48 B):
                const char *pk = reinterpret_cast<const char *>(w.wc + cid);      // in flight
                asm volatile("prefetch.global.L1 [%0];" :: "l"(pk));              // while the session closes
            }
            wbuf_advance(c, now);
            c.flags = (c.flags & ~WF_PHASE) | PH_FINISHED;
            if (S.records && c.session < sc.sess_cap) S.b->sess_flags[sc.sess_off + c.session] |= 1;
            wsync_session(w, c, now);
            wqoe_session(w, c, cid, true);
            c.flags &= ~(WF_LIVE | WF_OPEN);
            c.pc = C_SESSION;
            continue;
        case C_SEG_ERR:                                // OverloadError response
            if (c.attempt == sc.retries) {             // give up: the session is aborted (client.py:257-260)
                if (S.records && c.session < sc.sess_cap) S.b->sess_flags[sc.sess_off + c.session] |= 2;
                wsync_session(w, c, now);
                wqoe_session(w, c, cid, false);
                c.flags &= ~(WF_LIVE | WF_OPEN);
                c.pc = C_SESSION;
                continue;
            }
            delay = ldexp(sc.retry_backoff, c.attempt);
            next = C_RETRY;
            break;
        case C_RETRY:                                  // after sleep(backoff): backoff *= 2
            c.attempt++;
            if (S.records) w.wc[cid].requested = now;
            delay = w.L;
            next = C_SEG_LAT;
            break;
        default:
            return;
        }
        if (xfer) {
            // the trace samples, the period bits and the byte count load together
            const Trace tr = S.trace(cid);
            const TraceAhead a = trace_ahead(tr, trace_phase(tr, now));
            const int64_t nbytes = next == C_SEG_XFER ? (int64_t)(int32_t)S.size(wdesc(S, c)) : S.manifest(c.seq);
            size = nbytes;
            delay = completion_time_at(tr, a, now, nbytes) - now;
        }
        if (!arm(w, c, cid, now, delay, next)) return;
        if (next == C_SEG_LAT) { S.flag(OTF_S_INTERNAL); return; }   // zero latency never reaches this engine
    }
}

// one client event: state in registers for the whole chain
__device__ __forceinline__ void client_event(Win &w, int32_t cid, double when, int32_t path) {
    WClient c;
    load_client_stream(c, &w.cl[cid]);
    client_local_body(w, c, cid, path >= 0 ? when : c.next_when, path);
    store_client_stream(&w.cl[cid], c);
}

// SessionReport.harvest at the horizon (orchestrator.py:357-359, client.py:177-187)
__device__ __forceinline__ void wharvest(Win &w, WClient &c, int32_t cid, double horizon) {
    if (c.pc == C_HUNG) w.S.flag(OTF_S_HUNG);
    if (!(c.flags & WF_OPEN)) return;
    if (c.flags & WF_LIVE) {
        wbuf_advance(c, horizon);
        wsync_session(w, c, horizon);
    }
    wqoe_session(w, c, cid, false);
}

__device__ __forceinline__ int32_t warp_min(int32_t v) {
    v = __reduce_min_sync(0xffffffffu, v);
    return v;
}

// Order the window's server events by (time, arm time, client): each lane
// ranks its entries against all others (ties are flagged afterwards).
__device__ __forceinline__ bool key_gt(double wa, int32_t ia, double wb, int32_t ib) {
    return wa > wb || (wa == wb && ia > ib);
}

#ifndef WIN_NO_QSORT
// Fast rank sort of a window's n <= 32 E server events (lane l holds positions
// l, l + 32, ...): rank by a 32-bit fixed-point key q = (t - window start) *
// 2^32 / W, broadcast by shuffle.  q is monotone non-decreasing in t, so if the
// ranks form a permutation the order is the time order; equal keys collide,
// which the check after the scatter sees (a position left unwritten, or not
// strictly increasing: a tie).  Then the list is restored and false returned,
// and the exact sorts run.
template <int E>
__device__ __forceinline__ bool qsort_fast(Win &w, int lane, int32_t n) {
    double t[E];
    int16_t c[E];
    uint16_t d[E];
    int32_t p[E], r[E];
    uint32_t q[E];
    const double base = (double)w.k * w.W, scale = w.invW * 4294967296.0;
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        const bool v = i < n;
        t[e] = v ? w.lw[i] : INFINITY;
        c[e] = v ? w.li[i] : 0;
        d[e] = v ? w.ld[i] : 0;
        p[e] = v ? w.lp[i] : 0;
        const double x = (t[e] - base) * scale;
        q[e] = x <= 0.0 ? 0u : x >= 4294967295.0 ? 0xffffffffu : (uint32_t)x;
        r[e] = 0;
    }
#pragma unroll QSORT_UNROLL
    for (int32_t j = 0; j < n; j++) {
        uint32_t src = q[0];
#pragma unroll
        for (int e = 1; e < E; e++) src = (j >> 5) == e ? q[e] : src;
        const uint32_t qj = __shfl_sync(0xffffffffu, src, j & 31);
#pragma unroll
        for (int e = 0; e < E; e++) r[e] += (int32_t)(qj < q[e]);
    }
    __syncwarp();                                      // every lane has read the list
#pragma unroll
    for (int e = 0; e < E; e++)
        if (lane + 32 * e < n) w.lw[lane + 32 * e] = NAN;   // unwritten positions stay NaN
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++)
        if (lane + 32 * e < n) { w.lw[r[e]] = t[e]; w.li[r[e]] = c[e]; w.ld[r[e]] = d[e]; w.lp[r[e]] = p[e]; }
    __syncwarp();
    bool ok = true;                                    // strictly increasing, every position written
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        if (i < n) ok &= w.lw[i] == w.lw[i] && (i == 0 || w.lw[i] > w.lw[i - 1]);
    }
    if (__all_sync(0xffffffffu, ok)) return true;
    __syncwarp();                                      // collision or tie: restore the list
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        if (i < n) { w.lw[i] = t[e]; w.li[i] = c[e]; w.ld[i] = d[e]; w.lp[i] = p[e]; }
    }
    __syncwarp();
    return false;
}
#endif

#ifndef WIN_NO_BSORT
// Bucket sort of a window's n <= 32 E server events by the same 32-bit fixed-point key
// (list capacity >= 64 E: positions 32 E..64 E of the time array are its scratch):
// 32 E buckets on the key's top bits (shared-memory counters), a warp scan for their
// starts, then each event's rank within its bucket by comparing with the bucket's
// other keys (~1 on average).  ~1/3 of the rank sort's instructions.  The result and
// the check are the rank sort's: equal keys collide (fallback to the exact sorts).
template <int E>
__device__ __forceinline__ bool qsort_bucket(Win &w, int lane, int32_t n) {
    constexpr int NB = 32 * E, SH = E == 2 ? 26 : 25;
    static_assert(E == 2 || E == 4, "64 or 128 events");
    double t[E];
    int16_t c[E];
    uint16_t d[E];
    int32_t p[E], r[E];
    uint32_t q[E], bk[E], slot[E];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(w.lw + NB), *tq = cnt + NB;
    const double base = (double)w.k * w.W, scale = w.invW * 4294967296.0;
#pragma unroll
    for (int e = 0; e < E; e++) cnt[lane + 32 * e] = 0u;
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        const bool v = i < n;
        t[e] = v ? w.lw[i] : INFINITY;
        c[e] = v ? w.li[i] : 0;
        d[e] = v ? w.ld[i] : 0;
        p[e] = v ? w.lp[i] : 0;
        const double x = (t[e] - base) * scale;
        q[e] = x <= 0.0 ? 0u : x >= 4294967295.0 ? 0xffffffffu : (uint32_t)x;
        bk[e] = q[e] >> SH;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++)
        if (lane + 32 * e < n) slot[e] = atomicAdd(&cnt[bk[e]], 1u);
    __syncwarp();
    uint32_t cb[E], tot = 0;                           // lane: buckets E l .. E l + E - 1
#pragma unroll
    for (int e = 0; e < E; e++) { cb[e] = cnt[E * lane + e]; tot += cb[e]; }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    uint32_t run = incl - tot;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) { cnt[E * lane + e] = run | (cb[e] << 16); run += cb[e]; }   // start | count << 16
    __syncwarp();
    uint32_t st[E], nb[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        st[e] = 0; nb[e] = 0;
        if (lane + 32 * e < n) {
            const uint32_t sc = cnt[bk[e]];
            st[e] = sc & 0xffffu;
            nb[e] = sc >> 16;
            tq[st[e] + slot[e]] = q[e];
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) {
        int32_t rk = (int32_t)st[e];
        OTF_NOUNROLL
        for (uint32_t k = 0; k < nb[e]; k++) rk += (int32_t)(tq[st[e] + k] < q[e]);
        r[e] = rk;
    }
    __syncwarp();                                      // every lane has read the list
#pragma unroll
    for (int e = 0; e < E; e++)
        if (lane + 32 * e < n) w.lw[lane + 32 * e] = NAN;   // unwritten positions stay NaN
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++)
        if (lane + 32 * e < n) { w.lw[r[e]] = t[e]; w.li[r[e]] = c[e]; w.ld[r[e]] = d[e]; w.lp[r[e]] = p[e]; }
    __syncwarp();
    bool ok = true;                                    // strictly increasing, every position written
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        if (i < n) ok &= w.lw[i] == w.lw[i] && (i == 0 || w.lw[i] > w.lw[i - 1]);
    }
    if (__all_sync(0xffffffffu, ok)) return true;
    __syncwarp();                                      // collision or tie: restore the list
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = lane + 32 * e;
        if (i < n) { w.lw[i] = t[e]; w.li[i] = c[e]; w.ld[i] = d[e]; w.lp[i] = p[e]; }
    }
    __syncwarp();
    return false;
}
#endif

// Order the window's server events by time: rank sort for small windows, in-place
// bitonic sort for large ones.  Equal times are flagged afterwards; order_ties
// then orders each group by arm time, a result independent of the group's order.
// NW: warps per scenario of the calling kernel.  Two-warp kernels sort windows of more
// than RANK_SORT_MAX events with both warps (sort_bucket_cta / sort_list_cta), so
// their copy carries only the <= 64-event paths (hot code).
template <int NW>
__device__ void sort_list(Win &w, int lane) {
    WinHeader *h = w.h;
    const int32_t n = h->n_list;
    if (lane == 0) h->n_ties = 0;
    if (n <= 1) { __syncwarp(); return; }
#ifdef WIN_REG_SORT
    if (n <= 64) {
        // bitonic network over 64 positions in registers: lane holds positions lane and
        // lane + 32; keys are (time bit pattern, list position) -- non-negative doubles order
        // like their bit patterns, and the position breaks equal times (flagged below and
        // reordered by order_ties).  Then every lane gathers its two positions' payloads.
        const bool v0 = lane < n, v1 = lane + 32 < n;
        unsigned long long k0 = v0 ? (unsigned long long)__double_as_longlong(w.lw[lane]) : ~0ull;
        unsigned long long k1 = v1 ? (unsigned long long)__double_as_longlong(w.lw[lane + 32]) : ~0ull;
        int32_t j0 = lane, j1 = lane + 32;
        OTF_NOUNROLL
        for (int32_t size = 2; size <= 64; size <<= 1) {
            OTF_NOUNROLL
            for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride == 32) {                    // partner: the lane's other position
                    const bool sw = (k0 > k1) | ((k0 == k1) & (j0 > j1));   // size == 64: ascending
                    const unsigned long long tk = sw ? k1 : k0;
                    k1 = sw ? k0 : k1; k0 = tk;
                    const int32_t tj = sw ? j1 : j0;
                    j1 = sw ? j0 : j1; j0 = tj;
                } else {
                    const bool lower = (lane & stride) == 0;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        unsigned long long &k = h ? k1 : k0;
                        int32_t &j = h ? j1 : j0;
                        const unsigned long long pk = __shfl_xor_sync(0xffffffffu, k, stride);
                        const int32_t pj = __shfl_xor_sync(0xffffffffu, j, stride);
                        const bool asc = ((lane + 32 * h) & size) == 0 || size == 64;
                        const bool mine_gt = (k > pk) | ((k == pk) & (j > pj));
                        // keep the smaller key when this position is the lower one of an ascending pair
                        const bool take = (lower == asc) ? mine_gt : !mine_gt;
                        k = take ? pk : k;
                        j = take ? pj : j;
                    }
                }
            }
        }
        const int16_t c0 = v0 ? w.li[j0] : 0, c1 = v1 ? w.li[j1] : 0;
        const uint16_t d0 = v0 ? w.ld[j0] : 0, d1 = v1 ? w.ld[j1] : 0;
        const int32_t s0 = v0 ? w.lp[j0] : 0, s1 = v1 ? w.lp[j1] : 0;
        __syncwarp();                                  // every lane has read its payloads
        if (v0) { w.lw[lane] = __longlong_as_double((long long)k0); w.li[lane] = c0; w.ld[lane] = d0; w.lp[lane] = s0; }
        if (v1) { w.lw[lane + 32] = __longlong_as_double((long long)k1); w.li[lane + 32] = c1; w.ld[lane + 32] = d1; w.lp[lane + 32] = s1; }
        // equal request times (rare): neighbours in the sorted order
        const unsigned long long up0 = __shfl_up_sync(0xffffffffu, k0, 1);
        const unsigned long long last0 = __shfl_sync(0xffffffffu, k0, 31);
        const unsigned long long up1 = __shfl_up_sync(0xffffffffu, k1, 1);
        const bool tie = (lane > 0 && v0 && k0 == up0) || (v1 && k1 == (lane > 0 ? up1 : last0));
        const bool any = __any_sync(0xffffffffu, tie);
        if (lane == 0) h->n_ties = any ? 1 : 0;
        __syncwarp();
        return;
    }
#endif
#ifndef WIN_NO_QSORT
#ifndef WIN_QSORT_MAX
#define WIN_QSORT_MAX 128                              // fast rank sort up to this many events
#endif
    // (in the two-warp kernels warp 0 alone bucket-sorting 65-128 events measured -3% on
    // config 4 but +2% on c5t, profiles/r02i_ab_bsort*; they take sort_bucket_cta)
#ifndef WIN_NO_BSORT
    bool fast;
    if constexpr (NW == 1)
        fast = n <= 64 ? (h->list_cap >= 128 ? qsort_bucket<2>(w, lane, n) : qsort_fast<2>(w, lane, n))
                       : n <= WIN_QSORT_MAX &&
                             (h->list_cap >= 256 ? qsort_bucket<4>(w, lane, n) : qsort_fast<4>(w, lane, n));
    else
        fast = h->list_cap >= 128 ? qsort_bucket<2>(w, lane, n) : qsort_fast<2>(w, lane, n);
#else
    const bool fast = n <= 64 ? qsort_fast<2>(w, lane, n) : n <= WIN_QSORT_MAX && qsort_fast<4>(w, lane, n);
#endif
    if (fast) {
        if (lane == 0) h->n_ties = 0;
        __syncwarp();
        return;
    }
#endif
    if (n <= RANK_SORT_MAX) {
        // each lane ranks elements lane and lane + 32 in one pass over the list (one
        // broadcast load per j for both).  Non-negative doubles order like
        // their bit patterns, so the compares run on the integer pipe.
        const int32_t i0 = lane, i1 = lane + 32;
        const bool v0 = i0 < n, v1 = i1 < n;
        const double w0 = v0 ? w.lw[i0] : INFINITY, w1 = v1 ? w.lw[i1] : INFINITY;
        const int32_t id0 = v0 ? w.li[i0] : 0x7fff, id1 = v1 ? w.li[i1] : 0x7fff;
        const unsigned long long t0 = (unsigned long long)__double_as_longlong(w0);
        const unsigned long long t1 = (unsigned long long)__double_as_longlong(w1);
        const unsigned long long *lwb = reinterpret_cast<const unsigned long long *>(w.lw);
        int32_t r0 = 0, r1 = 0;
#pragma unroll SORT_UNROLL
        for (int32_t j = 0; j < n; j++) {              // branch-free (time, list position) compare:
            const unsigned long long tj = lwb[j];      //   equal times are flagged below and
            r0 += (int32_t)((tj < t0) | ((tj == t0) & (j < i0)));   //   reordered by order_ties,
            r1 += (int32_t)((tj < t1) | ((tj == t1) & (j < i1)));   //   whose result is order-free
        }
        const uint16_t d0 = v0 ? w.ld[i0] : 0, d1 = v1 ? w.ld[i1] : 0;
        const int32_t s0 = v0 ? w.lp[i0] : 0, s1 = v1 ? w.lp[i1] : 0;
        __syncwarp();                                  // every lane has read the list
        if (v0) { w.lw[r0] = w0; w.li[r0] = (int16_t)id0; w.ld[r0] = d0; w.lp[r0] = s0; }
        if (v1) { w.lw[r1] = w1; w.li[r1] = (int16_t)id1; w.ld[r1] = d1; w.lp[r1] = s1; }
        __syncwarp();
        // equal request times (rare): neighbours in the sorted list
        const bool tie = (i0 > 0 && v0 && w.lw[i0] == w.lw[i0 - 1]) || (v1 && w.lw[i1] == w.lw[i1 - 1]);
        const bool any = __any_sync(0xffffffffu, tie);
        if (lane == 0) h->n_ties = any ? 1 : 0;
        __syncwarp();
        return;
    } else if constexpr (NW == 1) {
        int32_t p = 1;
        while (p < n) p <<= 1;
        OTF_NOUNROLL
        for (int32_t i = n + lane; i < p; i += 32) { w.lw[i] = INFINITY; w.li[i] = 32767; }
        __syncwarp();
        for (int32_t size = 2; size <= p; size <<= 1) {
            for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
                OTF_NOUNROLL
                for (int32_t t = lane; t < (p >> 1); t += 32) {
                    int32_t lo = 2 * t - (t & (stride - 1));
                    int32_t hi = lo + stride;
                    bool up = (lo & size) == 0;
                    double wl = w.lw[lo], wh = w.lw[hi];
                    int32_t il = w.li[lo], ih = w.li[hi];
                    if (key_gt(wl, il, wh, ih) == up) {
                        w.lw[lo] = wh; w.lw[hi] = wl;
                        w.li[lo] = (int16_t)ih; w.li[hi] = (int16_t)il;
                        uint16_t td = w.ld[lo]; w.ld[lo] = w.ld[hi]; w.ld[hi] = td;
                        int32_t tp = w.lp[lo]; w.lp[lo] = w.lp[hi]; w.lp[hi] = tp;
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    bool tie = false;                                  // any equal request times? (rare)
    OTF_NOUNROLL
    for (int32_t i = lane + 1; i < n; i += 32) tie |= w.lw[i] == w.lw[i - 1];
    bool any = __any_sync(0xffffffffu, tie);
    if (lane == 0) h->n_ties = any ? 1 : 0;
    __syncwarp();
}

#ifndef WIN_NO_BSORT
// Two-warp bucket sort of a window's 64 < n <= 64 E server events (list capacity >=
// 128 E: positions 64 E..128 E of the time array are its scratch), the CTA version of
// qsort_bucket: thread t holds positions t, t + 64, ...; 64 E buckets on the 32-bit
// key's top bits; warp 0 scans the bucket counts.  Six CTA barriers instead of the
// bitonic sort's 28 (36) stages.  Returns false (list restored) on a key collision.
template <int E>
__device__ bool sort_bucket_cta(Win &w, int tid, int32_t m) {
    static_assert(E == 2 || E == 4, "128 or 256 events");
    constexpr int NB = 64 * E, SH = E == 2 ? 25 : 24, PL = NB / 32;
    WinHeader *h = w.h;
    const int32_t n = h->n_list;
    const int lane = tid & 31;
    double t[E];
    int16_t c[E];
    uint16_t d[E];
    int32_t p[E], r[E];
    uint32_t q[E], bk[E], slot[E];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(w.lw + NB), *tq = cnt + NB;
    const double base = (double)m * w.W, scale = w.invW * 4294967296.0;
#pragma unroll
    for (int e = 0; e < E; e++) cnt[tid + 64 * e] = 0u;
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = tid + 64 * e;
        const bool v = i < n;
        t[e] = v ? w.lw[i] : INFINITY;
        c[e] = v ? w.li[i] : 0;
        d[e] = v ? w.ld[i] : 0;
        p[e] = v ? w.lp[i] : 0;
        const double x = (t[e] - base) * scale;
        q[e] = x <= 0.0 ? 0u : x >= 4294967295.0 ? 0xffffffffu : (uint32_t)x;
        bk[e] = q[e] >> SH;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++)
        if (tid + 64 * e < n) slot[e] = atomicAdd(&cnt[bk[e]], 1u);
    __syncthreads();
    if (tid < 32) {                                    // warp 0: lane holds buckets PL l .. PL l + PL - 1
        uint32_t cb[PL], tot = 0;
#pragma unroll
        for (int e = 0; e < PL; e++) { cb[e] = cnt[PL * lane + e]; tot += cb[e]; }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t run = incl - tot;
        __syncwarp();
#pragma unroll
        for (int e = 0; e < PL; e++) { cnt[PL * lane + e] = run | (cb[e] << 16); run += cb[e]; }   // start | count << 16
    }
    __syncthreads();
    uint32_t st[E], nb[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        st[e] = 0; nb[e] = 0;
        if (tid + 64 * e < n) {
            const uint32_t sc = cnt[bk[e]];
            st[e] = sc & 0xffffu;
            nb[e] = sc >> 16;
            tq[st[e] + slot[e]] = q[e];
        }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++) {
        int32_t rk = (int32_t)st[e];
        OTF_NOUNROLL
        for (uint32_t k = 0; k < nb[e]; k++) rk += (int32_t)(tq[st[e] + k] < q[e]);
        r[e] = rk;
        if (tid + 64 * e < n) w.lw[tid + 64 * e] = NAN;    // unwritten positions stay NaN
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++)
        if (tid + 64 * e < n) { w.lw[r[e]] = t[e]; w.li[r[e]] = c[e]; w.ld[r[e]] = d[e]; w.lp[r[e]] = p[e]; }
    __syncthreads();
    bool ok = true;                                    // strictly increasing, every position written
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int32_t i = tid + 64 * e;
        if (i < n) ok &= w.lw[i] == w.lw[i] && (i == 0 || w.lw[i] > w.lw[i - 1]);
    }
    if (__syncthreads_and(ok ? 1 : 0)) {
        if (tid == 0) h->n_ties = 0;
        __syncthreads();
        return true;
    }
#pragma unroll
    for (int e = 0; e < E; e++) {                      // collision or tie: restore the list
        const int32_t i = tid + 64 * e;
        if (i < n) { w.lw[i] = t[e]; w.li[i] = c[e]; w.ld[i] = d[e]; w.lp[i] = p[e]; }
    }
    __syncthreads();
    return false;
}
#endif

// Two-warp bitonic sort of a large window's list (NW = 2: the big client classes,
// e.g. ~180 requests per window at 10,000 clients): both warps take the
// compare-exchanges of every stage, a CTA barrier between stages.  Called by all
// threads after the window selection; the result and the tie flag are the same
// as sort_list's.
__device__ void sort_list_cta(Win &w, int tid, int nthreads) {
    WinHeader *h = w.h;
    const int32_t n = h->n_list;
    int32_t p = 1;
    while (p < n) p <<= 1;
    OTF_NOUNROLL
    for (int32_t i = n + tid; i < p; i += nthreads) { w.lw[i] = INFINITY; w.li[i] = 32767; }
    __syncthreads();
    for (int32_t size = 2; size <= p; size <<= 1) {
        for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
            OTF_NOUNROLL
            for (int32_t t = tid; t < (p >> 1); t += nthreads) {
                const int32_t lo = 2 * t - (t & (stride - 1));
                const int32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double wl = w.lw[lo], wh = w.lw[hi];
                const int32_t il = w.li[lo], ih = w.li[hi];
                if (key_gt(wl, il, wh, ih) == up) {
                    w.lw[lo] = wh; w.lw[hi] = wl;
                    w.li[lo] = (int16_t)ih; w.li[hi] = (int16_t)il;
                    const uint16_t td = w.ld[lo]; w.ld[lo] = w.ld[hi]; w.ld[hi] = td;
                    const int32_t tp = w.lp[lo]; w.lp[lo] = w.lp[hi]; w.lp[hi] = tp;
                }
            }
            __syncthreads();
        }
    }
    bool tie = false;                                  // any equal request times? (rare)
    OTF_NOUNROLL
    for (int32_t i = tid + 1; i < n; i += nthreads) tie |= w.lw[i] == w.lw[i - 1];
    const int any = __syncthreads_or(tie ? 1 : 0);
    if (tid == 0) h->n_ties = any ? 1 : 0;
    __syncthreads();
}

// Equal request times (rare): order each tie group by arm time (the tick order
// of their latency timers, sim.py:304-309); equal arm times cannot be ordered.
__device__ void order_ties(Win &w) {
    WinHeader *h = w.h;
    const int32_t n = h->n_list;
    for (int32_t i = 1; i < n; i++) {
        if (w.lw[i] != w.lw[i - 1]) continue;
        int32_t j = i;                                 // insertion step by ctime
        while (j > 0 && w.lw[j] == w.lw[j - 1]) {
            double cj = req_ctime(w, w.li[j]), cp = req_ctime(w, w.li[j - 1]);
            if (cj == cp) { atomicOr(&h->st.status, OTF_S_TIE); break; }
            if (cj > cp) break;
            int16_t ti = w.li[j]; w.li[j] = w.li[j - 1]; w.li[j - 1] = ti;
            uint16_t td = w.ld[j]; w.ld[j] = w.ld[j - 1]; w.ld[j - 1] = td;
            int32_t tp = w.lp[j]; w.lp[j] = w.lp[j - 1]; w.lp[j - 1] = tp;
            j--;
        }
    }
}

// Next non-empty window after k_done on the wheel (warp-wide bitmap scan).
__device__ int32_t wheel_next(WinHeader *h, int32_t k_done, int lane) {
    const int32_t start = k_done + 1;
    const int32_t p0 = start & (RING - 1);
    const int32_t w0 = p0 >> 5;
    constexpr int32_t NW = RING / 32;
    int32_t best = WIN_NONE;
    // virtual words 0..NW: word 0 = first word from bit p0, word NW = its low bits (wrap)
    for (int32_t v = lane; v <= NW; v += 32) {
        uint32_t bits;
        if (v == 0) bits = h->bits[w0] & (0xffffffffu << (p0 & 31));
        else if (v == NW) bits = (p0 & 31) ? (h->bits[w0] & ((1u << (p0 & 31)) - 1)) : 0u;
        else bits = h->bits[(w0 + v) & (NW - 1)];
        if (bits) {
            int32_t slot = (((v == NW ? w0 : (w0 + v) & (NW - 1))) << 5) + (__ffs(bits) - 1);
            int32_t dist = (slot - p0) & (RING - 1);
            if (v == NW && dist == 0) dist = RING;
            best = min(best, start + dist);
        }
    }
    return warp_min(best);
}

#ifndef WIN_NO_PF_RESP
// Warm L2 with what the request's response chain reads in phase B (a cache hit
// answers at the request's own arrival time): the client's hot state, the trace
// sample the transfer starts in, the trace's period bits and the segment size.
// Issued by all lanes at the window's gather, ~15 k cycles before phase B
// (measured: -0.9% on the config-5 sweep, profiles/r02f_ab_redux_prefetch.txt).
__device__ __forceinline__ void prefetch_response(const Win &w, const SrvEnt &e) {
    const Scn &S = w.S;
    asm volatile("prefetch.global.L2 [%0];" :: "l"(w.cl + e.cid));
    asm volatile("prefetch.global.L2 [%0];" :: "l"(S.sizes + e.desc));
    if (S.sc->off_tr_i < 0) {
        const double q = e.when * S.inv_grid_step;
        const int32_t i = q < (double)S.sc->n_samples ? (int32_t)q : 0;
        asm volatile("prefetch.global.L2 [%0];" :: "l"(S.values + (int64_t)e.cid * S.sc->n_samples + i));
        asm volatile("prefetch.global.L2 [%0];" :: "l"(S.pbits + e.cid));
    }
}
#endif

// status bits that end a scenario's run early (the host re-runs it)
#define WIN_ABORT_BITS (OTF_S_TIE | OTF_S_UNFIT | OTF_S_LIST_OVERFLOW)

// Window-loop control word (shared): what both warps do after the selection step.
enum { CTL_RUN = 0, CTL_REFILE = 1, CTL_STOP = 2 };

// Two warps per scenario.  Warp 0 selects the next window, pops its buckets and
// sorts the server events; then, concurrently, lane 0 of warp 0 replays the
// server events (phase A) while warp 1 runs the window's client-local timers
// (clients with a local timer due are never touched by phase A: they are not
// waiting on the backend and have no pending request).  Finally both warps run
// the clients phase A responded to.
// NW warps per scenario.  NW = 1: 7 CTAs per SM run 1,024 config-5 scenarios on
// 148 SMs in one wave; the register file is split over the 4 SM sub-partitions
// (16 k each), so two-warp CTAs at that occupancy would cap the kernel at 128
// registers.  NW = 2 serves the shared-memory classes that fit at most 4 CTAs
// per SM anyway (10,000-client scenarios): 8 warps per SM keep ~240 registers.
// MB: resident CTAs per SM the register budget is sized for.  Two-warp CTAs come
// in two budgets: 4 per SM (up to 256 registers: the big shared-memory classes and
// sparse launches) and 7 per SM (14 warps on 4 sub-partitions: 128 registers, so a
// 1,024-scenario sweep stays one wave; measured 755 vs 785 ms for one warp).
template <bool RECORDS, int NW, int MB>
__global__ void __launch_bounds__(32 * NW, MB) windowed_kernel(const otf_batch b) {
    constexpr int WIN_WARPS = NW, WIN_THREADS = 32 * NW;
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    long long t_start = 0, t0 = 0, t1 = 0;
#ifdef WIN_BULK_GATHER
    uint32_t gphase = 0;                               // the gather mbarrier's phase parity (warp 0)
#endif
    const int32_t s = b.order ? b.order[blockIdx.x] : (int32_t)blockIdx.x;
    WinHeader *h = (WinHeader *)smem;
    if (tid == 0) { h->b = b; h->sc = b.scenarios[s]; }
    __syncthreads();
    Win w;
    w.S.init(&h->b, &h->sc, s);
    w.S.records = RECORDS;                             // compile-time: histogram kernels carry no record code
    const otf_scenario &sc = h->sc;
    const int32_t N = sc.n_clients, K = sc.n_workers;
    const int64_t D = (int64_t)sc.n_seq * sc.n_ranks * sc.max_nseg;
    uint8_t *p = smem + ((sizeof(WinHeader) + 15) & ~(size_t)15);
    const int32_t lcap = win_list_cap_sc(sc);
    w.lw = (double *)p; p += 8 * (int64_t)lcap;
    w.lp = (int32_t *)p; p += 4 * (int64_t)lcap;
    w.li = (int16_t *)p; p += 2 * (int64_t)lcap;
    w.ld = (uint16_t *)p; p += 2 * (int64_t)lcap;
    uint8_t *g = b.scratch + sc.scratch_off;
    WinGlobalLayout L = win_global_layout(N, D);
    w.h = h;
    w.bnext = (int16_t *)p; p += 2 * (int64_t)N;
    p = (uint8_t *)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    w.dflags = (uint16_t *)p;
    w.lstamp = (uint32_t *)(g + L.lstamp);
    w.lq = (LqEnt *)(g + L.lq);
    w.cl = (WPacked *)(g + L.clients);
    w.wc = (WCold *)(g + L.picks);
    w.S.cold = nullptr;                                // the exact engine's cold state (unused here)
    w.blist = (RespMsg *)(g + L.blist);
    w.bsrv = (SrvEnt *)(g + L.bsrv);
    w.bloc = (int32_t *)(g + L.bloc);
    w.scap = bucket_cap_srv(N);
    w.lcap = bucket_cap_loc(N);
    w.jq = (JobEnt *)(g + L.jobq);
    w.sq = (JobEnt *)(g + L.specq);
    // counters, QoE and small tables live in shared memory
    w.S.st = &h->st;
    w.S.stats = h->stats;
    w.S.qa = &h->qa;
    w.W = sc.latency * (1.0 - 0x1p-20);
    w.invW = 1.0 / w.W;
    w.H = sc.horizon;
    w.L = sc.latency;
    w.target = sc.target;
    w.k = -1;

    // ---- init -------------------------------------------------------------------
    const bool fits = win_fits(sc);
    const bool seq_smem = sc.n_seq <= MAXTAB;          // larger catalogs read their tables from global
    if (tid == 0) {
        EngineState z = {};
        z.lru_head = z.lru_tail = -1;
        h->st = z;
        for (int i = 0; i < OTF_ST_NSLOTS; i++) h->stats[i] = 0;
        qoe_zero(&h->qa, 0, 1);
        h->gq_head = 0; h->gq_n = K; h->fq_head = 0; h->fq_n = 0;
        h->jq_head = 0; h->jq_n = 0; h->jq_cap = (int32_t)(D + 1);
        h->sq_head = 0; h->sq_n = 0; h->tokens = 0;
        h->n_list = 0; h->n_blist = 0; h->wseq = 0;
        h->far_head = -1; h->far_n = 0; h->far_min = WIN_NONE; h->k_done = -1;
        h->arr_next = 0;
        h->arr_win = (fits && N > 0) ? timer_win(w, w.S.arrival(0)) : WIN_NONE;   // W > 0 only if fits
        h->ovf_head = -1; h->ovf_n = 0; h->ovf_min = WIN_NONE; h->n_loc = 0;
        h->lq_head = 0; h->lq_tail = 0; h->lq_stamp = 0; h->lq_cap = (int32_t)lq_capacity(D);
        h->list_cap = lcap;
#ifdef WIN_BULK_GATHER
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&h->gbar)));
#endif
        h->ctl = CTL_RUN; h->cur_m = 0;
        if (!fits) h->st.status |= OTF_S_UNFIT;        // not for this engine: host re-runs it exactly
    }
    __syncthreads();
    if (!fits) goto done;
    for (int32_t q = tid; q < MAXK; q += WIN_THREADS) {
        h->gq[q] = q;                                  // workers register as getters in id order
        WWorker z = {};
        z.win = WIN_NONE; z.pc = W_GOT; z.desc = -1; z.job = -1;
        h->wk[q] = z;
    }
    for (int32_t i = tid; i < RING / 2; i += WIN_THREADS) { h->cnt_srv[i] = 0; h->cnt_loc[i] = 0; }
    for (int32_t i = tid; i < RING / 32; i += WIN_THREADS) h->bits[i] = 0;
    for (int32_t i = tid; seq_smem && i < sc.n_seq; i += WIN_THREADS) {
        h->t_segcount[i] = w.S.segcounts[i];
        h->t_seqdur[i] = w.S.seqdur[i];
        h->t_segdur[i] = w.S.segdur[i];
        h->t_zipf[i] = w.S.zipf[i];
        h->t_manifest[i] = w.S.manifest_b[i];
    }
    for (int32_t i = tid; i < sc.n_ranks; i += WIN_THREADS) {
        h->t_rho[i] = w.S.rho[i];
        h->t_bitrates[i] = w.S.bitrates[i];
    }
    for (int64_t d = tid; d < D; d += WIN_THREADS) {
        w.lstamp[d] = 0; w.dflags[d] = DF_IDLE;
    }
    __syncthreads();
    if (seq_smem) {
        w.S.segcounts = h->t_segcount;
        w.S.seqdur = h->t_seqdur;
        w.S.segdur = h->t_segdur;
        w.S.zipf = h->t_zipf;
        w.S.manifest_b = h->t_manifest;
    }
    w.S.rho = h->t_rho;
    w.S.bitrates = h->t_bitrates;
    // clients: the first step arms sleep(offset) (orchestrator.py:337); offsets are a
    // cumulative sum, so clients join the wheel in id order (arrival cursor below)
    for (int32_t c = tid; c < N; c += WIN_THREADS) {
        WClient cl = {};
        double off = w.S.arrival(c);
        cl.pc = C_ARRIVED;
        cl.next_when = 0.0 + off;
        cl.session = -1;
        cl.est = -1.0;
        w.cl[c] = wpack(cl);
        if (!(off > 0)) w.S.flag(OTF_S_TIE);           // instant start: tick order among clients matters
        // the client's pick stream (orchestrator.py:338-340), seeded here in parallel rather
        // than by one lane at the arrival: it is first drawn from after the arrival
        seed_picks(&w.wc[c].picks, sc.seed, c);
    }
    __syncthreads();
    if (h->st.status & WIN_ABORT_BITS) goto done;

    // ---- window loop --------------------------------------------------------------
    t_start = clock64();
    if (tid == 0) server_begin(w);
    {
        // hand-offs are safe in the parallel server pass if no transcode can end inside
        // the window it starts in: svc >= svc_floor * (1 + min eps) >= 2 W
        double emin = sc.noise > 0 ? INFINITY : 0.0;
        if (sc.noise > 0)
            for (int64_t q = tid; q < (int64_t)K * sc.eps_stride; q += WIN_THREADS) emin = fmin(emin, w.S.eps[q]);
        for (int o = 16; o > 0; o >>= 1) emin = fmin(emin, __shfl_xor_sync(0xffffffffu, emin, o));
        if (lane == 0) h->wmin[warp] = emin;             // every warp's partial minimum
        __syncthreads();
        if (tid == 0) {
            for (int q = 1; q < WIN_WARPS; q++) emin = fmin(emin, h->wmin[q]);
            h->hand_safe = (w.svc_floor * (1.0 + emin) >= 2.0 * w.W) ? 1 : 0;
        }
        __syncthreads();
    }
    for (;;) {
        if (warp == 0) {
            t0 = WCLOCK();
            // next window: wheel, far list, worker timers, next arrival
            int32_t m = wheel_next(h, h->k_done, lane);
            int32_t mw = lane < K ? h->wk[lane].win : WIN_NONE;
            m = min(m, warp_min(mw));
            m = min(m, h->far_min);
            int32_t arr_win = WIN_NONE;
            arr_win = h->arr_win;
            m = min(m, arr_win);
            int32_t ctl = CTL_RUN;
            if (m == WIN_NONE) {
                ctl = CTL_STOP;
            } else {
#ifndef WIN_SERIAL_ARRIVALS
                if (arr_win != WIN_NONE && arr_win - m < RING / 2) {   // arrivals entering the wheel:
                    // a batch of ~RING/2 windows' worth, 32 clients at a time (offsets are a
                    // cumulative sum, so the clients that fit form a prefix of each chunk)
                    w.k = m - 1;                           // windows before m are empty: wheel base = m
                    int32_t base = h->arr_next;
                    for (;;) {
                        const int32_t c = base + lane;
                        const int32_t wk = c < N ? timer_win(w, w.S.arrival(c)) : WIN_NONE;
                        const bool ok = wk != WIN_NONE && wk - w.k < RING;
                        if (ok) bucket_push(w, c, wk, false, wunpack(w.cl[c]), 0.0, 0);
                        const int32_t got = __popc(__ballot_sync(0xffffffffu, ok));
                        base += got;
                        if (got < 32) break;
                    }
                    __syncwarp();                          // every lane has read arr_win / arr_next
                    if (lane == 0) {
                        h->k_done = m - 1;
                        h->arr_next = base;
                        h->arr_win = base < N ? timer_win(w, w.S.arrival(base)) : WIN_NONE;
                    }
                    __syncwarp();
                }
#else
                if (arr_win != WIN_NONE && arr_win - m < RING) {   // arrivals entering the wheel
                    if (lane == 0) {
                        h->k_done = m - 1;                 // windows before m are empty: wheel base = m
                        w.k = m - 1;
                        int32_t c = h->arr_next;
                        while (c < N) {
                            int32_t wk = timer_win(w, w.S.arrival(c));
                            if (wk == WIN_NONE || wk - w.k >= RING) break;   // wheel base is m - 1 here
                            bucket_push(w, c, wk, false, wunpack(w.cl[c]), 0.0, 0);
                            c++;
                        }
                        h->arr_next = c;
                        h->arr_win = c < N ? timer_win(w, w.S.arrival(c)) : WIN_NONE;
                    }
                    __syncwarp();
                }
#endif
                if (h->far_n > 0 && h->far_min < m + RING / 2) {   // far timers close to the wheel: re-file
                    if (lane == 0) {
                        int32_t c = h->far_head;
                        h->far_head = -1; h->far_n = 0; h->far_min = WIN_NONE;
                        h->k_done = m - 1;                 // windows before m are empty: wheel base = m
                        w.k = m - 1;
                        while (c >= 0) {
                            int32_t nx = w.bnext[c];
                            const WClient cl = wunpack(w.cl[c]);
                            const bool srv = cl.pc == C_SEG_LAT;
                            bucket_push(w, c, timer_win(w, cl.next_when), srv, cl, srv ? w.wc[c].ctime : 0.0,
                                        srv ? wdesc(w.S, cl) : 0);
                            c = nx;
                        }
                    }
                    __syncwarp();
                    ctl = CTL_REFILE;
                }
            }
            if (ctl == CTL_RUN) {
                w.k = m;
                w.E = (double)(m + 1) * w.W;
                if (h->lq_tail - h->lq_head > (uint32_t)(h->lq_cap / 4 * 3)) lq_compact_warp(w, lane);
                // pop the buckets: the window's arrays are read by all lanes at once
                const int32_t slot = m & (RING - 1);
                const uint32_t csh = (slot & 1) << 4;
                const int32_t ns = min((int32_t)((h->cnt_srv[slot >> 1] >> csh) & 0xffffu), w.scap);
                const int32_t nl = min((int32_t)((h->cnt_loc[slot >> 1] >> csh) & 0xffffu), w.lcap);
                int32_t n_ovf = 0, nb = 0;
                if (h->ovf_n > 0 && h->ovf_min <= m) {     // overflowed pushes due now (rare)
                    if (lane == 0) {
                        int32_t c = h->ovf_head, keep = -1, rem = WIN_NONE, kept = 0;
                        while (c >= 0) {
                            int32_t nx = w.bnext[c];
                            const WClient cl = wunpack(w.cl[c]);
                            int32_t wk = timer_win(w, cl.next_when);
                            if (wk == m) {
                                if (cl.pc == C_SEG_LAT) { if (ns + n_ovf < h->list_cap) w.li[ns + n_ovf] = (int16_t)c; n_ovf++; }
                                else { RespMsg lm; lm.when = cl.next_when; lm.cid = c; lm.path = -1; w.blist[nb++] = lm; }
                            } else {
                                w.bnext[c] = (int16_t)keep; keep = c; kept++;
                                rem = min(rem, wk);
                            }
                            c = nx;
                        }
                        h->ovf_head = keep; h->ovf_n = kept; h->ovf_min = rem;
                        h->n_list = ns + n_ovf;
                        h->n_blist = nb;
                    }
                    __syncwarp();
                    n_ovf = h->n_list - ns;
                    nb = h->n_blist;
                }
                const int32_t nlist = ns + n_ovf;
                if (nlist > h->list_cap) {                 // more simultaneous requests than the list holds:
                    if (lane == 0) atomicOr(&h->st.status, OTF_S_LIST_OVERFLOW);   // re-run with a larger one
                    ctl = CTL_STOP;
                } else {
                    const SrvEnt *as_g = w.bsrv + (int64_t)slot * w.scap;
                    const SrvEnt *as = as_g;
#ifdef WIN_BULK_GATHER
                    // the bucket (ns x 24 B, contiguous) into the list's free second half by
                    // one bulk copy (TMA engine, mbarrier completion), then read from shared
                    if (ns > 0 && ns <= 64 && h->list_cap >= 128) {
                        SrvEnt *stage = reinterpret_cast<SrvEnt *>(w.lw + 64);
                        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&h->gbar);
                        if (lane == 0) {
                            const uint32_t bytes = ((uint32_t)ns * (uint32_t)sizeof(SrvEnt) + 15u) & ~15u;
                            asm volatile("fence.proxy.async;" ::: "memory");
                            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
                            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                         :: "r"((uint32_t)__cvta_generic_to_shared(stage)), "l"(as), "r"(bytes), "r"(bar) : "memory");
                        }
                        uint32_t done = 0;
                        while (!done)
                            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                         : "=r"(done) : "r"(bar), "r"(gphase) : "memory");
                        gphase ^= 1u;
                        as = stage;
                    }
#endif
                    OTF_NOUNROLL
                    for (int32_t i = lane; i < ns; i += 64) {      // gather sort keys + request descriptors
                        const SrvEnt e = as[i];                    //   (both loads issue before the stores)
                        const bool two = i + 32 < ns;
                        SrvEnt f;
                        if (two) f = as[i + 32];
#ifndef WIN_NO_PF_RESP
                        prefetch_response(w, e);
                        if (two) prefetch_response(w, f);
#endif
                        w.li[i] = e.cid;
                        w.lw[i] = e.when;
                        w.ld[i] = e.desc;
                        w.lp[i] = e.pk;
                        if (two) { w.li[i + 32] = f.cid; w.lw[i + 32] = f.when; w.ld[i + 32] = f.desc; w.lp[i + 32] = f.pk; }
                    }
#ifdef WIN_NEXT_PF                                   // (measured -1.5% without it, profiles/r02q_abn_prefetch_flags.txt)
                    {                                      // warm L2 with the next window's request entries
                        const int32_t sn = (m + 1) & (RING - 1);
                        const int32_t nn = min((int32_t)((h->cnt_srv[sn >> 1] >> ((sn & 1) << 4)) & 0xffffu), w.scap);
                        if (8 * lane < nn)
                            asm volatile("prefetch.global.L2 [%0];" :: "l"(w.bsrv + (int64_t)sn * w.scap + 8 * lane));
                    }
#endif
                    OTF_NOUNROLL
                    for (int32_t i = ns + lane; i < nlist; i += 32) {   // overflowed pushes: from the client state
                        const int32_t c = w.li[i];
                        const WClient cl = wunpack(w.cl[c]);
                        w.lw[i] = cl.next_when;
                        w.ld[i] = (uint16_t)wdesc(w.S, cl);
                        w.lp[i] = (int32_t)cl.rank | ((int32_t)cl.index << 8) | ((int32_t)cl.seq << 16);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        h->stats[OTF_ST_WINDOWS]++;
                        h->cnt_srv[slot >> 1] &= ~(0xffffu << csh);
                        h->cnt_loc[slot >> 1] &= ~(0xffffu << csh);
                        h->bits[slot >> 5] &= ~(1u << (slot & 31));
                        h->n_list = nlist;
                        h->n_bsrv = ns;
                        h->n_blist = nb;
                        h->n_loc = nl;
                        h->cur_m = m;
                    }
                    __syncwarp();
                    t1 = WCLOCK();
                    if (lane == 0) h->stats[OTF_ST_CYC_SCAN] += t1 - t0;
                    t0 = t1;
                    if (WIN_WARPS == 1 || nlist <= RANK_SORT_MAX) {   // else both warps, below
                        sort_list<WIN_WARPS>(w, lane);
                        t1 = WCLOCK();
                        if (lane == 0) h->stats[OTF_ST_CYC_SORT] += t1 - t0;
                    }
                }
            }
            if (lane == 0) h->ctl = ctl;
        }
        __syncthreads();
        const int32_t ctl = h->ctl;
        if (ctl == CTL_STOP) break;
        if (ctl == CTL_REFILE) continue;
        if constexpr (WIN_WARPS == 2) {
            if (h->n_list > RANK_SORT_MAX) {           // a large window: both warps sort it
                t0 = WCLOCK();
#ifndef WIN_NO_BSORT
                const int32_t nl = h->n_list, lc = h->list_cap;
                bool done;
                if constexpr (MB <= 4)                 // the big classes' shape: up to 256 events
                    done = nl <= 128 ? lc >= 256 && sort_bucket_cta<2>(w, tid, h->cur_m)
                                     : nl <= 256 && lc >= 512 && sort_bucket_cta<4>(w, tid, h->cur_m);
                else                                   // (the dense shape: 12 B of spills with both)
                    done = nl <= 128 && lc >= 256 && sort_bucket_cta<2>(w, tid, h->cur_m);
                if (!done)
#endif
                    sort_list_cta(w, tid, WIN_THREADS);
                if (tid == 0) h->stats[OTF_ST_CYC_SORT] += WCLOCK() - t0;
            }
        }
        const int32_t m = h->cur_m;
        w.k = m;
        w.E = (double)(m + 1) * w.W;
        t0 = WCLOCK();
        // thread 0 = the server lane; with two warps, warp 1 runs the local timers meanwhile
        {
            // ---- phase A: the server events (the whole warp in request-only windows) ----
            int par = 0;
#ifdef WIN_DIAG
            long long dgp = clock64();
#endif
            int32_t pre = 0;
#ifndef WIN_SERIAL_PAR_OK
            if (warp == 0) {                           // warp-uniform answer
                par = parallel_ok(w) ? 1 : 0;
#ifndef WIN_NO_PREFIX
                if (!par && lane == 0) pre = parallel_prefix(w);
#endif
            }
#else
            if (tid == 0) {
                par = parallel_ok(w) ? 1 : 0;
#ifndef WIN_NO_PREFIX
                if (!par) pre = parallel_prefix(w);
#endif
            }
#endif
#ifdef WIN_DIAG
            if (tid == 0) h->stats[30] += clock64() - dgp;
#endif
            if (warp == 0) {
#ifdef WIN_SERIAL_PAR_OK
                par = __shfl_sync(0xffffffffu, par, 0);
#endif
                pre = __shfl_sync(0xffffffffu, pre, 0);
            }
            // one call site each (phase_a_parallel is inlined; a second copy of it, or a
            // non-inlined phase_a taking `w` by reference, costs hot code / a stack frame)
            if (warp == 0 && (par | pre)) {
                const int32_t n_all = h->n_list;
                __syncwarp();
                if (pre && lane == 0) h->n_list = pre;     // the prefix before the completion
                __syncwarp();
                phase_a_parallel(w, lane);
                if (pre && lane == 0) h->n_list = n_all;
            }
            if (tid == 0 && !par) {                    // the serial lane (after a parallel prefix)
                if (!pre && h->n_ties) order_ties(w);
                phase_a(w, pre);
            }
            if (tid == 0) {
                h->k_done = m;
                h->stats[OTF_ST_CYC_SERVER] += WCLOCK() - t0;
                if (par) h->stats[OTF_ST_PAR_WINDOWS]++;
            }
        }
        if constexpr (WIN_WARPS == 1) {
            // ---- phase B: the window's local timers, then the clients phase A responded
            // to, in ONE loop: a single inlined copy of the client state machine ----
            __syncwarp();
            t0 = WCLOCK();
            const int32_t nl = h->n_loc, nb = h->n_blist;
            const int32_t *al = w.bloc + (int64_t)(m & (RING - 1)) * w.lcap;
            // software-pipelined: the next event's client state is loaded (into registers)
            // while this one runs -- each client appears once per window and client events
            // touch only their own client, so the early load cannot be stale
            const int32_t total = nl + nb;
            int32_t i = lane;
            RespMsg nm;
            WClient nc;
            if (i < total) {
                if (i < nb) nm = w.blist[i]; else { nm.cid = al[i - nb]; nm.path = -1; }
                load_client_stream(nc, &w.cl[nm.cid]);
            }
            while (i < total) {
                const RespMsg m = nm;
                WClient c = nc;
                i += 32;
                if (i < total) {
                    if (i < nb) nm = w.blist[i]; else { nm.cid = al[i - nb]; nm.path = -1; }
                    load_client_stream(nc, &w.cl[nm.cid]);
                }
                client_local_body(w, c, m.cid, m.path >= 0 ? m.when : c.next_when, m.path);
                store_client_stream(&w.cl[m.cid], c);
            }
            __syncwarp();
            if (h->st.status & WIN_ABORT_BITS) break;
        } else {
            // ---- phase B1: warp 1 runs the window's client-local timers, concurrent with
            // phase A; then (B2) both warps run the clients phase A responded to (and the
            // overflowed local timers).  One loop, so ONE inlined copy of the client state
            // machine (hot code); its trip counts are warp-uniform, so the CTA barrier
            // between the stages is reached convergently ----
            const int32_t *al = w.bloc + (int64_t)(m & (RING - 1)) * w.lcap;
            const long long tb = clock64();
            int32_t n_items = warp > 0 ? h->n_loc : 0, base = 0, step = 32;
            bool b2 = false, abort = false;
            for (;;) {
                if (base >= n_items) {
                    if (b2) break;
                    if (warp > 0 && lane == 0) h->stats[OTF_ST_CYC_LOCAL] += clock64() - tb;
                    __syncthreads();
                    if (h->st.status & WIN_ABORT_BITS) { abort = true; break; }
                    t0 = WCLOCK();
                    b2 = true;
                    n_items = h->n_blist;
                    base = 32 * warp;
                    step = WIN_THREADS;
                    continue;
                }
                const int32_t i = base + lane;
                base += step;
                if (i < n_items) {
                    RespMsg msg;
                    if (b2) msg = w.blist[i]; else { msg.cid = al[i]; msg.when = 0.0; msg.path = -1; }
                    client_event(w, msg.cid, msg.when, msg.path);
                }
            }
            if (abort) break;
            __syncthreads();
        }
        if (tid == 0) h->stats[OTF_ST_CYC_CLIENTS] += WCLOCK() - t0;
    }
    if (tid == 0) {
        server_end(w);
        h->stats[OTF_ST_CYC_TOTAL] += clock64() - t_start;
    }

    // ---- horizon: harvest (orchestrator.py:357-359) ----
    if (!(h->st.status & WIN_ABORT_BITS)) {
        for (int32_t c = tid; c < N; c += WIN_THREADS) {
            WClient cl = wunpack(w.cl[c]);
            wharvest(w, cl, c, sc.horizon);
        }
    }
    __syncthreads();
done:
    if (tid == 0) {
        int64_t *gs = b.stats + (int64_t)s * OTF_ST_NSLOTS;
        h->stats[OTF_ST_CACHE_CAPACITY] = sc.cache_capacity;
        h->stats[OTF_ST_CURRENT_BYTES] = h->st.cur_bytes;
        h->stats[OTF_ST_ENTRIES] = h->st.entries;
        h->stats[OTF_ST_STATUS] = h->st.status;
        for (int i = 0; i < OTF_ST_NSLOTS; i++) gs[i] = h->stats[i];
        int64_t *cnt = b.counts + (int64_t)s * 4;
        cnt[0] = h->st.n_req; cnt[1] = h->st.n_sess; cnt[2] = h->st.n_seg; cnt[3] = h->st.n_job;
        b.status[s] = h->st.status;
    }
    __syncthreads();
    if (tid == 0) w.S.flush_qoe();                     // the summary pass completes the block
}

}  // namespace otf

int64_t otf_windowed_scratch_bytes(int32_t n_clients, int32_t n_workers, int64_t n_desc) {
    (void)n_workers;
    return otf::win_global_layout(n_clients, n_desc).total;
}

bool otf_windowed_fits(const otf_scenario &sc) { return otf::win_fits(sc); }

int64_t otf_windowed_shared_bytes(int32_t n_clients, int64_t n_desc, int32_t list_cap) {
    return otf::win_smem_bytes(n_clients, n_desc, list_cap > 0 ? list_cap : otf::win_list_cap(n_clients));
}

int32_t otf_windowed_list_cap(int32_t n_clients) { return otf::win_list_cap(n_clients); }

// Kernel shape per launch: 1 = one warp per scenario (8 per SM); 2 = two warps,
// 256-register budget (4 per SM); 3 = two warps, 128-register budget (7 per SM).
// Two warps once shared memory allows at most 4 CTAs per SM, or once at most 4
// scenarios per SM are resident anyway (a strong-scaling shard: the second warp
// runs the window's local timers during the server pass and the responded
// clients take one round); the 7-per-SM two-warp budget while the launch (with
// the launches running beside it) fits 7 per SM in one wave; else one warp.
// OTF_WIN_NW=1|2|3 overrides the choice (A/B measurements).
static int windowed_shape(const otf_batch &b) {
    const int smem = (int)b.shared_bytes;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int32_t resident = b.concurrent > b.n_scenarios ? b.concurrent : b.n_scenarios;
    int shape = 1;
    if ((smem + 1024) * 5 > 228 * 1024 || resident <= 4 * sms) shape = 2;
    else if (resident <= 7 * sms && (smem + 1024) * 7 <= 228 * 1024) shape = 3;
    if (const char *e = getenv("OTF_WIN_NW")) {
        const int v = atoi(e);
        if (v >= 1 && v <= 3) shape = v;
    }
    return shape;
}

int otf_launch_windowed(const otf_batch &b, cudaStream_t stream) {
    int smem = (int)b.shared_bytes;
    const int shape = windowed_shape(b);
    const int nw = shape == 1 ? 1 : 2;
    auto kern = b.mode == OTF_MODE_RECORDS
                    ? (shape == 1 ? otf::windowed_kernel<true, 1, 8>
                                  : shape == 2 ? otf::windowed_kernel<true, 2, 4> : otf::windowed_kernel<true, 2, 7>)
                    : (shape == 1 ? otf::windowed_kernel<false, 1, 8>
                                  : shape == 2 ? otf::windowed_kernel<false, 2, 4> : otf::windowed_kernel<false, 2, 7>);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return 1;
    }
    if (const char *e = getenv("OTF_WIN_CARVEOUT"))    // A/B: shared-memory carveout in percent (L1 size)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
    kern<<<b.n_scenarios, 32 * nw, smem, stream>>>(b);
    return 0;
}
