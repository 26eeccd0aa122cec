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
    unsigned long long acc[XACC_LIMBS];
    uint32_t flags;
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
    const int64_t n_req = q->n_requests, nt = q->n_lat_tail, ns = q->n_stall_tail;
    const double *lat = b.tail_lat ? b.tail_lat + sc.lat_off : nullptr;
    const otf_stall_ent *ent = b.tail_stall ? b.tail_stall + sc.stl_off : nullptr;
    if ((nt > 0 && !lat) || (ns > 0 && !ent)) return;   // no tails: no order statistics

    if (tid < XACC_LIMBS) S.acc[tid] = 0;
    if (tid == 0) S.flags = 0;
    __syncthreads();
    // ---- exact latency sum ----
    for (int64_t i = tid; i < nt; i += SUM_THREADS) xacc_add(S.acc, lat[i], &S.flags);

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
            for (int64_t i = tid; i < nt; i += SUM_THREADS) {
                const unsigned long long v = (unsigned long long)__double_as_longlong(lat[i]);
                const uint32_t dg = (uint32_t)(v >> lo) & mask;
                const bool top = hi == 63;
                if (!done[0] && (top || (v >> (hi + 1)) == (p0 >> (hi + 1)))) atomicAdd(&S.hist[0][dg], 1u);
                if (!done[1] && (top || (v >> (hi + 1)) == (p1 >> (hi + 1)))) atomicAdd(&S.hist[1][dg], 1u);
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

    // ---- stall sum in registration order ----
    otf_stall_ent *sorted = b.tail_stall + sc.stl_off + sc.stl_cap;
    for (int64_t base = 0; base < ns; base += (int64_t)SUM_THREADS * PER_THREAD) {
        unsigned long long mk[PER_THREAD];
        long long ms[PER_THREAD];
        int64_t cnt[PER_THREAD];
#pragma unroll
        for (int k = 0; k < PER_THREAD; k++) {
            const int64_t i = base + tid + (int64_t)k * SUM_THREADS;
            mk[k] = i < ns ? (unsigned long long)__double_as_longlong(ent[i].reg_time) : ~0ull;
            ms[k] = i < ns ? ent[i].sid : 0;
            cnt[k] = 0;
        }
        for (int64_t t0 = 0; t0 < ns; t0 += TILE) {
            __syncthreads();
            for (int j = tid; j < TILE; j += SUM_THREADS) {
                if (t0 + j < ns) {
                    S.tkey[j] = (unsigned long long)__double_as_longlong(ent[t0 + j].reg_time);
                    S.tsid[j] = ent[t0 + j].sid;
                }
            }
            __syncthreads();
            const int m = (int)min((int64_t)TILE, ns - t0);
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
            if (i < ns) sorted[cnt[k]] = ent[i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        double total = 0.0;                            // sum() of the np.float64 stall times
        bool tie = false;
        unsigned long long prev = ~0ull;
        for (int64_t i = 0; i < ns; i++) {
            const otf_stall_ent e = sorted[i];
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
        q->stall_time_sum = total;
        q->latency_sum = xacc_round(S.acc);
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
