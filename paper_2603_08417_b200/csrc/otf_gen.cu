// otf_gen.cu -- request generation on the device: the reference's seeded numpy
// streams replayed by the GPU (include/otfgpu.h otf_gen_tables).
//
// Every stream the reference draws per run comes from its own
// Generator(PCG64(SeedSequence(entropy))):
//   * trace  c: standard_normal(n + 1) from SS([seed, 2, c]), turned into
//     bandwidth samples x' = mu + (x - mu) * decay + spread * z,
//     bw = min(max(exp(x), floor), cap) (netem.py:179-202), then the period
//     bits sum(v * width) (netem.py:61-64, CPython 3.12 compensated sum);
//   * arrivals: cumsum(exponential(1 / rate, N)) from SS([seed, 1])
//     (orchestrator.py:265-268; np.cumsum is sequential);
//   * worker w's noise: normal(0, noise) from SS([seed, w]) (transcode.py:89-99).
// One thread replays one stream, in the stream's own order, with the
// arithmetic of otf_npdist.cuh (numpy 2.3.5's ziggurats) and otf_libm.cuh
// (glibc's exp / log1p): the tables are bit-identical to the host replicas in
// otf_hostgen.cu, which tests/test_host.py pins against numpy itself.
//
// Cost model: a config-5 sweep needs 64 x 2,800 traces of 601 draws (1.1e8
// draws, 0.86 GB of samples written once) plus 64 arrival and 256 noise
// streams.  Traces are spread one per thread over every SM; a trace thread
// buffers 16 samples per row in shared memory and writes them as whole
// 128-byte lines, so the rows go out coalesced instead of one 8-byte store
// per row per step.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <string>

#include "otf_npdist.cuh"
#include "otfgpu.h"

namespace otf {

constexpr int GEN_THREADS = 128;
constexpr int GEN_CHUNK = 16;                          // samples per row flushed at once (one 128-byte line)

__device__ __forceinline__ void seed_stream3(Pcg64 &g, uint64_t a, uint64_t b, uint64_t c, int n) {
    uint32_t w[8];
    int m = 0;
    m = push_words(w, m, a);
    m = push_words(w, m, b);
    if (n > 2) m = push_words(w, m, c);
    pcg_seed(g, w, m);
}

__device__ int find_job(const otf_gen_job *jobs, int n_jobs, int64_t t) {
    int lo = 0, hi = n_jobs - 1;                       // last job with first_stream <= t
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].first_stream <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// One trace per thread.  The block's rows are staged GEN_CHUNK samples at a
// time in shared memory ([chunk][thread], conflict-free) and flushed as whole
// lines: after every chunk the block writes its rows' 128-byte segments, lane
// by lane, so each warp store covers four full lines.
__device__ void gen_trace(const otf_gen_job &J, int64_t c, bool active, double *pool, double (*stage)[GEN_THREADS],
                          int64_t row0, int rows) {
    Pcg64 g;
    double x = 0.0;
    PySum pb;
    const double *starts = pool + J.off_starts;
    double *values = pool + J.off_out;
    if (active) {
        seed_stream3(g, J.seed, 2, (uint64_t)c, 3);
        x = J.mu + J.sigma * np_standard_normal(g);
    }
    const int n = J.n;
    for (int i0 = 0; i0 < n; i0 += GEN_CHUNK) {
        const int m = min(GEN_CHUNK, n - i0);
        if (active) {
            for (int k = 0; k < m; k++) {
                const int i = i0 + k;
                const double e = libm::exp(x);
                double bw = e > J.floor_bps ? e : J.floor_bps;
                bw = J.cap_bps < bw ? J.cap_bps : bw;
                stage[k][threadIdx.x] = bw;
                const double end = (i + 1 < n) ? starts[i + 1] : J.period;
                pb.add(bw * (end - starts[i]));
                x = J.mu + (x - J.mu) * J.decay + J.spread * np_standard_normal(g);
            }
        }
        __syncthreads();
        // flush: row r's samples [i0, i0 + m) are contiguous in values
        for (int e = threadIdx.x; e < rows * m; e += GEN_THREADS) {
            const int r = e / m, k = e - r * m;
            values[(row0 + r) * (int64_t)n + i0 + k] = stage[k][r];
        }
        __syncthreads();
    }
    if (active) pool[J.off_pbits + c] = pb.result();
}

// Every job starts on a block boundary (the host rounds first_stream up to a
// multiple of GEN_THREADS), so a block belongs to exactly one job.
__global__ void __launch_bounds__(GEN_THREADS) gen_kernel(const otf_gen_job *jobs, int32_t n_jobs, double *pool) {
    __shared__ double stage[GEN_CHUNK][GEN_THREADS];
    const int64_t t0 = (int64_t)blockIdx.x * GEN_THREADS;
    const otf_gen_job &J = jobs[find_job(jobs, n_jobs, t0)];
    const int64_t row0 = t0 - J.first_stream;
    if (row0 >= J.n_streams) return;                   // padding between jobs (whole block)
    const int64_t s = row0 + threadIdx.x;
    if (J.kind == OTF_GEN_TRACE) {
        const int64_t left = J.n_streams - row0;
        const int rows = left < GEN_THREADS ? (int)left : GEN_THREADS;
        gen_trace(J, s, s < J.n_streams, pool, stage, row0, rows);
        return;
    }
    if (s >= J.n_streams) return;
    Pcg64 g;
    if (J.kind == OTF_GEN_ARRIVALS) {
        seed_stream3(g, J.seed, 1, 0, 2);
        double *out = pool + J.off_out;
        double acc = 0.0;
        for (int i = 0; i < J.n; i++) {
            acc += J.scale * np_standard_exponential(g);
            out[i] = acc;
        }
    } else if (J.kind == OTF_GEN_NOISE) {
        seed_stream3(g, J.seed, (uint64_t)s, 0, 2);
        double *out = pool + J.off_out + s * (int64_t)J.n;
        for (int i = 0; i < J.n; i++) out[i] = 0.0 + J.scale * np_standard_normal(g);
    }
}

__global__ void libm_kernel(int32_t fn, const double *x, int64_t n, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = fn == 0 ? libm::exp(x[i]) : libm::log1p(x[i]);
}

}  // namespace otf

int otf_fail(int code, const std::string &msg);

extern "C" {

int otf_gen_tables(const otf_gen_job *jobs_dev, int32_t n_jobs, int64_t total_streams, double *f64_pool,
                   void *stream) {
    if (n_jobs < 0 || total_streams < 0 || (n_jobs > 0 && (!jobs_dev || !f64_pool)))
        return otf_fail(OTF_EINVAL, "otf_gen_tables: bad arguments");
    if (n_jobs == 0 || total_streams == 0) return OTF_OK;
    const int64_t blocks = (total_streams + otf::GEN_THREADS - 1) / otf::GEN_THREADS;
    otf::gen_kernel<<<(unsigned)blocks, otf::GEN_THREADS, 0, (cudaStream_t)stream>>>(jobs_dev, n_jobs, f64_pool);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? OTF_OK : otf_fail(OTF_ECUDA, std::string("otf_gen_tables: ") + cudaGetErrorString(e));
}

int otf_model_libm(int32_t fn, const double *x, int64_t n, double *out) {
    if (n < 0 || (n > 0 && (!x || !out)) || (fn != 0 && fn != 1)) return otf_fail(OTF_EINVAL, "otf_model_libm: bad arguments");
    for (int64_t i = 0; i < n; i++) out[i] = fn == 0 ? otf::libm::exp(x[i]) : otf::libm::log1p(x[i]);
    return OTF_OK;
}

int otf_model_libm_dev(int32_t fn, const double *x, int64_t n, double *out, void *stream) {
    if (n < 0 || (n > 0 && (!x || !out)) || (fn != 0 && fn != 1))
        return otf_fail(OTF_EINVAL, "otf_model_libm_dev: bad arguments");
    if (n == 0) return OTF_OK;
    otf::libm_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(fn, x, n, out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? OTF_OK : otf_fail(OTF_ECUDA, std::string("otf_model_libm_dev: ") + cudaGetErrorString(e));
}

}  // extern "C"
