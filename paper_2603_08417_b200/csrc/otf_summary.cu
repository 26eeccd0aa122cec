// otf_summary.cu -- the summary pass: completes each scenario's otf_qoe from
// the engines' summary tails, so ExperimentResult.summary()
// (orchestrator.py:280-309, metrics.py:67-116) is exact without per-request
// records.  One CTA per scenario, after either engine, on the same stream:
//
//   latency_p50 / latency_p99   sorted(latencies)[n // 2] and
//                               [min(n - 1, int(0.99 * n))] (orchestrator.py:297-299).
//                               Zero latencies (storage / cache hits) are only
//                               counted; the nonzero ones sit in the tail and a
//                               two-rank radix select (11-bit digits over the
//                               IEEE bit patterns, which order like the values
//                               for non-negative doubles) finds both ranks.
//   latency_sum                 exact sum of the tail (otf_xacc.cuh) == math.fsum
//   stall_hist / n_stalls /     from the closed-session records the engines append
//   n_finished                  (one atomic and one store per session close)
//   startup_delay_sum           exact sum of the startup-delay tail == math.fsum
//   stall_time_sum              stalls_per_session's sum (metrics.py:88-92): the
//                               stalled sessions ordered by (registration time,
//                               session id) and added left to right, as CPython
//                               adds the np.float64 stall times in registration
//                               order.  The windowed engine numbers sessions in
//                               parallel, so two stalled sessions registered at
//                               the identical instant have no known order: the
//                               scenario is flagged OTF_S_TIE (exact-engine re-run).
#include <cuda_runtime.h>
#include <stdint.h>

#include "otf_state.cuh"
#include "otfgpu.h"

namespace otf {

constexpr int SUM_THREADS = 512;
constexpr int SEL_BITS = 11, SEL_BINS = 1 << SEL_BITS;
constexpr int TILE = 1024;                     // stall-sort key tile (shared)
constexpr int PER_THREAD = 4;                  // stall entries ranked per thread per round
constexpr int32_t RERUN = OTF_S_TIE | OTF_S_UNFIT | OTF_S_TAIL_OVERFLOW | OTF_S_EPS_OVERFLOW | OTF_S_INTERNAL;

struct SumShared {
    unsigned long long acc[XACC_LIMBS];        // exact latency sum
    unsigned long long sup[XACC_LIMBS];        // exact startup-delay sum
    unsigned long long priv[SUM_THREADS][XACC_LIMBS];   // per-thread limbs (no atomic contention)
    uint32_t flags;
    uint32_t stall_hist[OTF_STALL_BINS];
    unsigned long long n_stalls;
    uint32_t n_finished, n_stl;
    uint32_t hist[2][SEL_BINS];
    unsigned long long tkey[TILE];             // registration-time bits
    long long tsid[TILE];
    unsigned long long pre[2];                 // selected prefix per rank
    long long rem[2];                          // rank within the candidates sharing the prefix
};

__device__ __forceinline__ bool key_less(unsigned long long ka, long long sa, unsigned long long kb, long long sb) {
    return ka < kb || (ka == kb && sa < sb);
}

__global__ void __launch_bounds__(SUM_THREADS) summary_kernel(const otf_batch b, int32_t engine) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    SumShared &S = *reinterpret_cast<SumShared *>(sm_raw);
    const int s = b.order ? b.order[blockIdx.x] : (int)blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const otf_scenario &sc = b.scenarios[s];
    otf_qoe *q = b.qoe + s;
    if (b.status[s] & RERUN) return;                   // the host re-runs this scenario
    if (!b.tail_lat || !b.tail_sess || !b.tail_sup) return;
    const int64_t n_req = q->n_requests, nt = q->n_lat_tail, ns = q->n_sessions, nsup = q->n_started;
    const double *lat = b.tail_lat + sc.lat_off;
    const otf_sess_ent *ses = b.tail_sess + sc.ses_off;
    otf_sess_ent *stl = b.tail_sess + sc.ses_off + sc.ses_cap;      // stalled sessions, gathered
    otf_sess_ent *sorted = stl + sc.stl_cap;                        //   ... and in registration order
    const double *sup = b.tail_sup + sc.sup_off;

    for (int i = tid; i < OTF_STALL_BINS; i += SUM_THREADS) S.stall_hist[i] = 0;
    if (tid == 0) { S.flags = 0; S.n_stalls = 0; S.n_finished = 0; S.n_stl = 0; }
    __syncthreads();
    // ---- exact sums of the latencies and startup delays: each thread adds into its
    //      own limb row (values of one scenario share their exponents, so shared
    //      atomics would all hit the same words), then the rows are summed ----
    for (int pass = 0; pass < 2; pass++) {
        const double *v = pass ? sup : lat;
        const int64_t n = pass ? nsup : nt;
        unsigned long long *row = S.priv[tid];
#pragma unroll
        for (int i = 0; i < XACC_LIMBS; i++) row[i] = 0;
        bool bad = false;
        for (int64_t i = tid; i < n; i += SUM_THREADS) {
            int qq;
            uint32_t c0, c1, c2;
            if (!xacc_split(v[i], qq, c0, c1, c2)) { bad = true; continue; }
            row[qq] += c0; row[qq + 1] += c1; row[qq + 2] += c2;
        }
        if (bad) atomicOr(&S.flags, XACC_INEXACT);
        __syncthreads();
        if (tid < XACC_LIMBS) {                        // column sums: < 2^32 terms of < 2^33 each
            unsigned long long t = 0;
            for (int r = 0; r < SUM_THREADS; r++) t += S.priv[r][tid];
            (pass ? S.sup : S.acc)[tid] = t;
        }
        __syncthreads();
    }
    // ---- the session records: stall histogram, finished count, stall events; the
    //      stalled sessions gathered for the ordered sum ----
    {
        unsigned long long my_stalls = 0;
        uint32_t my_fin = 0, my_zero = 0;              // most sessions never stall: bin 0 in a register
        for (int64_t base = 0; base < ns; base += SUM_THREADS) {
            const int64_t i = base + tid;
            otf_sess_ent e;
            e.stall_time = 0.0; e.stalls = 0;
            if (i < ns) {
                e = ses[i];
                const uint32_t st = e.stalls & ~OTF_SE_FINISHED;
                my_fin += e.stalls >> 31;
                my_stalls += st;
                if (st == 0) my_zero++;
                else atomicAdd(&S.stall_hist[st < OTF_STALL_BINS - 1 ? st : OTF_STALL_BINS - 1], 1u);
            }
            const bool stalled = i < ns && e.stall_time != 0.0;   // gathered: one atomic per warp
            const unsigned m = __ballot_sync(0xffffffffu, stalled);
            uint32_t pos0 = 0;
            if (lane == 0 && m) pos0 = atomicAdd(&S.n_stl, (uint32_t)__popc(m));
            pos0 = __shfl_sync(0xffffffffu, pos0, 0);
            if (stalled) {
                const uint32_t pos = pos0 + __popc(m & ((1u << lane) - 1u));
                if (pos < (uint64_t)sc.stl_cap) stl[pos] = e;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            my_stalls += __shfl_xor_sync(0xffffffffu, my_stalls, o);
            my_fin += __shfl_xor_sync(0xffffffffu, my_fin, o);
            my_zero += __shfl_xor_sync(0xffffffffu, my_zero, o);
        }
        if (lane == 0) {
            atomicAdd(&S.n_stalls, my_stalls);
            atomicAdd(&S.n_finished, my_fin);
            atomicAdd(&S.stall_hist[0], my_zero);
        }
    }
    __syncthreads();
    const int64_t nstl = S.n_stl;
    if (nstl > sc.stl_cap) {                           // more stalled sessions than room: re-run
        if (tid == 0) {
            q->n_stall_tail = nstl;
            b.status[s] |= OTF_S_TAIL_OVERFLOW;
            b.stats[(int64_t)s * OTF_ST_NSLOTS + OTF_ST_STATUS] |= OTF_S_TAIL_OVERFLOW;
        }
        return;
    }

    // ---- order statistics: ranks n // 2 and min(n - 1, int(0.99 n)) of all latencies ----
    const int64_t k50 = n_req / 2;
    const int64_t k99 = n_req > 0 ? min(n_req - 1, (int64_t)(0.99 * (double)n_req)) : 0;
    const int64_t zeros = n_req - nt;                  // latency 0.0 sorts first
    bool done[2];
    done[0] = n_req == 0 || k50 < zeros;
    done[1] = n_req == 0 || k99 < zeros;
    if (tid == 0) {
        S.pre[0] = S.pre[1] = 0;
        S.rem[0] = k50 - zeros;
        S.rem[1] = k99 - zeros;
    }
    if (!(done[0] && done[1])) {
        for (int hi = 63; hi >= 0; hi -= SEL_BITS) {
            const int lo = hi - (SEL_BITS - 1) > 0 ? hi - (SEL_BITS - 1) : 0;
            const uint32_t mask = (1u << (hi - lo + 1)) - 1u;
            for (int i = tid; i < 2 * SEL_BINS; i += SUM_THREADS) (&S.hist[0][0])[i] = 0;
            __syncthreads();
            const unsigned long long p0 = S.pre[0], p1 = S.pre[1];
            const bool top = hi == 63;
            for (int64_t base = 0; base < nt; base += SUM_THREADS) {   // lanes with equal digits add once
                const int64_t i = base + tid;
                const unsigned long long v = i < nt ? (unsigned long long)__double_as_longlong(lat[i]) : 0ull;
#pragma unroll
                for (int r = 0; r < 2; r++) {
                    const unsigned long long p = r ? p1 : p0;
                    const bool in = i < nt && !done[r] && (top || (v >> (hi + 1)) == (p >> (hi + 1)));
                    const int dg = in ? (int)((uint32_t)(v >> lo) & mask) : -1;
                    const unsigned peers = __match_any_sync(0xffffffffu, dg);
                    if (in && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&S.hist[r][dg], (uint32_t)__popc(peers));
                }
            }
            __syncthreads();
            if (warp < 2 && !done[warp]) {             // warp r finds the digit holding rank r
                const int r = warp;
                const int per = SEL_BINS / 32;
                uint32_t mine = 0;
                for (int k = 0; k < per; k++) mine += S.hist[r][lane * per + k];
                uint32_t x = mine;                     // inclusive warp scan
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const long long want = S.rem[r];
                const unsigned hit = __ballot_sync(0xffffffffu, (long long)x > want);
                const int L = __ffs(hit) - 1;          // first lane whose prefix passes the rank
                __syncwarp();                          // every lane has read S.rem[r]
                if (lane == L) {
                    long long below = (long long)(x - mine);
                    int bin = lane * per;
                    while (below + (long long)S.hist[r][bin] <= want) { below += S.hist[r][bin]; bin++; }
                    S.pre[r] |= (unsigned long long)bin << lo;
                    S.rem[r] = want - below;
                }
            }
            __syncthreads();
            if (lo == 0) break;
        }
    }
    __syncthreads();

    // ---- stall sum in registration order: rank each stalled session by
    //      (registration time, session id) against tiles of all of them ----
    for (int64_t base = 0; base < nstl; base += (int64_t)SUM_THREADS * PER_THREAD) {
        unsigned long long mk[PER_THREAD];
        long long ms[PER_THREAD];
        int64_t cnt[PER_THREAD];
#pragma unroll
        for (int k = 0; k < PER_THREAD; k++) {
            const int64_t i = base + tid + (int64_t)k * SUM_THREADS;
            mk[k] = i < nstl ? (unsigned long long)__double_as_longlong(stl[i].reg_time) : ~0ull;
            ms[k] = i < nstl ? stl[i].sid : 0;
            cnt[k] = 0;
        }
        for (int64_t t0 = 0; t0 < nstl; t0 += TILE) {
            __syncthreads();
            for (int j = tid; j < TILE; j += SUM_THREADS) {
                if (t0 + j < nstl) {
                    S.tkey[j] = (unsigned long long)__double_as_longlong(stl[t0 + j].reg_time);
                    S.tsid[j] = stl[t0 + j].sid;
                }
            }
            __syncthreads();
            const int m = (int)min((int64_t)TILE, nstl - t0);
            for (int j = 0; j < m; j++) {
                const unsigned long long kj = S.tkey[j];
                const long long sj = S.tsid[j];
#pragma unroll
                for (int k = 0; k < PER_THREAD; k++) cnt[k] += key_less(kj, sj, mk[k], ms[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < PER_THREAD; k++) {
            const int64_t i = base + tid + (int64_t)k * SUM_THREADS;
            if (i < nstl) sorted[cnt[k]] = stl[i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        double total = 0.0;                            // sum() of the np.float64 stall times
        bool tie = false;
        unsigned long long prev = ~0ull;
        for (int64_t i = 0; i < nstl; i++) {
            const otf_sess_ent e = sorted[i];
            const unsigned long long k = (unsigned long long)__double_as_longlong(e.reg_time);
            tie |= k == prev;
            prev = k;
            total += e.stall_time;
        }
        if (tie && engine == OTF_ENGINE_WINDOWED) {    // registration order unknown: exact-engine re-run
            b.status[s] |= OTF_S_TIE;
            b.stats[(int64_t)s * OTF_ST_NSLOTS + OTF_ST_STATUS] |= OTF_S_TIE;
            return;
        }
        for (int i = 0; i < OTF_STALL_BINS; i++) q->stall_hist[i] = S.stall_hist[i];
        q->n_stalls = (int64_t)S.n_stalls;
        q->n_finished = S.n_finished;
        q->n_stall_tail = nstl;
        q->stall_time_sum = total;
        q->latency_sum = xacc_round(S.acc);
        q->startup_delay_sum = xacc_round(S.sup);
        q->latency_p50 = done[0] ? 0.0 : __longlong_as_double((long long)S.pre[0]);
        q->latency_p99 = done[1] ? 0.0 : __longlong_as_double((long long)S.pre[1]);
        q->summary_flags |= OTF_Q_ORDER_STATS | S.flags;
    }
}

}  // namespace otf

int otf_launch_summary(const otf_batch &b, int32_t engine, cudaStream_t stream) {
    const int smem = (int)sizeof(otf::SumShared);
    if (cudaFuncSetAttribute(otf::summary_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return 1;
    otf::summary_kernel<<<b.n_scenarios, otf::SUM_THREADS, smem, stream>>>(b, engine);
    return 0;
}
