// otf_capi.cu -- the extern "C" boundary of libotfgpu.so (include/otfgpu.h).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "otf_state.cuh"
#include "otfgpu.h"

int otf_launch_exact(const otf_batch &b, cudaStream_t stream);
int otf_launch_windowed(const otf_batch &b, cudaStream_t stream);
int otf_launch_summary(const otf_batch &b, int32_t engine, cudaStream_t stream);
int64_t otf_windowed_scratch_bytes(int32_t n_clients, int32_t n_workers, int64_t n_desc);
int64_t otf_windowed_shared_bytes(int32_t n_clients, int64_t n_desc, int32_t list_cap);
int32_t otf_windowed_list_cap(int32_t n_clients);
bool otf_windowed_fits(const otf_scenario &sc);
int otf_launch_sizes(const otf_size_table *tables_dev, int32_t n_tables, int64_t *i64_pool,
                     const double *f64_pool, const int32_t *i32_pool, cudaStream_t stream);

static thread_local std::string g_last_error;

static int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int otf_fail(int code, const std::string &msg) { return fail(code, msg); }   // for otf_hostgen.cu

static int check_cuda(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(OTF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return OTF_OK;
}

namespace {
// A Trace over caller pointers (host or device), as Scn::trace() builds it.
__host__ __device__ inline otf::Trace model_trace(const double *starts, const double *values, int32_t n,
                                                   double period, double pbits, double grid) {
    otf::Trace t;
    t.starts = starts; t.values = values; t.n = n;
    t.period = period; t.pbits = pbits; t.grid = grid;
    t.inv_grid = grid > 0 ? 1.0 / grid : 0.0;
    return t;
}

__global__ void model_completion_kernel(const double *starts, const double *values, int32_t n_samples,
                                        double period, double pbits, double grid, const double *start,
                                        const int64_t *nbytes, int32_t n, double *out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        out[i] = otf::completion_time(model_trace(starts, values, n_samples, period, pbits, grid), start[i], nbytes[i]);
}
}  // namespace

extern "C" {

int otf_version(void) { return OTF_ABI_VERSION; }

double otf_model_completion_time(const double *starts, const double *values, int32_t n, double period, double pbits,
                                 double grid, double start, int64_t nbytes) {
    return otf::completion_time(model_trace(starts, values, n, period, pbits, grid), start, nbytes);
}

int32_t otf_model_select_quality(double level, int32_t cur, int32_t has_est, double est, const int64_t *bitrates,
                                 int32_t top, double panic, double safe, double headroom) {
    return otf::select_quality(level, cur, has_est != 0, est, bitrates, top, panic, safe, headroom);
}

int otf_model_buffer_run(double t0, int32_t n, const int32_t *op, const double *t, const double *dur, double startup,
                         double resume, double *out) {
    if (n < 0 || (n > 0 && (!op || !t || !dur || !out))) return fail(OTF_EINVAL, "otf_model_buffer_run: bad arguments");
    otf::Buffer b;
    otf::buf_reset(b, t0);
    for (int32_t i = 0; i < n; i++) {
        if (op[i]) otf::buf_on_segment(b, t[i], dur[i], startup, resume);
        else otf::buf_advance(b, t[i]);
        double *o = out + 6 * (int64_t)i;
        o[0] = b.level; o[1] = b.phase; o[2] = b.stall_events; o[3] = b.stall_time; o[4] = b.started_at;
        o[5] = b.last_sync;
    }
    return OTF_OK;
}

int otf_model_exact_sum(const double *v, int64_t n, double *out) {
    if (!out || (n > 0 && !v)) return fail(OTF_EINVAL, "otf_model_exact_sum: bad arguments");
    unsigned long long limb[otf::XACC_LIMBS] = {};
    int inexact = 0;
    for (int64_t i = 0; i < n; i++) {
        int q;
        uint32_t c0, c1, c2;
        if (!otf::xacc_split(v[i], q, c0, c1, c2)) { inexact = 1; continue; }
        limb[q] += c0; limb[q + 1] += c1; limb[q + 2] += c2;
    }
    *out = otf::xacc_round(limb);
    return inexact;
}

int otf_model_completion_times(const double *starts, const double *values, int32_t n_samples, double period,
                               double pbits, double grid, const double *start, const int64_t *nbytes, int32_t n,
                               double *out, void *stream) {
    if (n < 0 || n_samples <= 0 || (n > 0 && (!starts || !values || !start || !nbytes || !out)))
        return fail(OTF_EINVAL, "otf_model_completion_times: bad arguments");
    if (n == 0) return OTF_OK;
    model_completion_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(starts, values, n_samples, period,
                                                                               pbits, grid, start, nbytes, n, out);
    return check_cuda("otf_model_completion_times");
}

const char *otf_last_error(void) { return g_last_error.c_str(); }

size_t otf_sizeof_scenario(void) { return sizeof(otf_scenario); }
size_t otf_sizeof_batch(void) { return sizeof(otf_batch); }
size_t otf_sizeof_qoe(void) { return sizeof(otf_qoe); }

int64_t otf_scratch_bytes(int32_t engine, int32_t n_clients, int32_t n_workers, int32_t n_seq,
                          int32_t n_ranks, int32_t max_nseg) {
    int64_t n_desc = (int64_t)n_seq * n_ranks * max_nseg;
    if (engine == OTF_ENGINE_WINDOWED) return otf_windowed_scratch_bytes(n_clients, n_workers, n_desc);
    return otf::exact_layout(n_clients, n_workers, n_desc).total;
}

int32_t otf_engine_fits(int32_t engine, const otf_scenario *sc) {
    if (!sc) return 0;
    if (engine == OTF_ENGINE_WINDOWED) return otf_windowed_fits(*sc) ? 1 : 0;
    return engine == OTF_ENGINE_EXACT ? 1 : 0;
}

int64_t otf_shared_bytes(int32_t engine, int32_t n_clients, int32_t n_workers, int32_t n_seq,
                         int32_t n_ranks, int32_t max_nseg) {
    (void)n_workers;
    if (engine != OTF_ENGINE_WINDOWED) return 0;
    return otf_windowed_shared_bytes(n_clients, (int64_t)n_seq * n_ranks * max_nseg, 0);
}

int64_t otf_shared_bytes_cap(int32_t n_clients, int32_t n_seq, int32_t n_ranks, int32_t max_nseg, int32_t list_cap) {
    return otf_windowed_shared_bytes(n_clients, (int64_t)n_seq * n_ranks * max_nseg, list_cap);
}

int32_t otf_list_cap(int32_t n_clients) { return otf_windowed_list_cap(n_clients); }

int otf_gen_sizes(const otf_size_table *tables_dev, int32_t n_tables, int64_t total_entries,
                  int64_t *i64_pool, const double *f64_pool, const int32_t *i32_pool, void *stream) {
    (void)total_entries;
    if (n_tables < 0 || (n_tables > 0 && (!tables_dev || !i64_pool || !f64_pool || !i32_pool)))
        return fail(OTF_EINVAL, "otf_gen_sizes: bad arguments");
    otf_launch_sizes(tables_dev, n_tables, i64_pool, f64_pool, i32_pool, (cudaStream_t)stream);
    return check_cuda("otf_gen_sizes");
}

int otf_run_batch(const otf_batch *batch, int32_t engine, void *stream) {
    if (!batch) return fail(OTF_EINVAL, "otf_run_batch: null batch");
    const otf_batch &b = *batch;
    if (b.n_scenarios < 0) return fail(OTF_EINVAL, "otf_run_batch: negative scenario count");
    if (b.n_scenarios == 0) return OTF_OK;
    if (!b.scenarios || !b.f64_pool || !b.i64_pool || !b.i32_pool || !b.scratch || !b.counts || !b.stats ||
        !b.qoe || !b.status)
        return fail(OTF_EINVAL, "otf_run_batch: missing device buffer");
    if (b.mode == OTF_MODE_RECORDS && (!b.req_id || !b.sess_client || !b.seg_session || !b.job_seq))
        return fail(OTF_EINVAL, "otf_run_batch: records mode needs record buffers");
    cudaStream_t s = (cudaStream_t)stream;
    if (engine == OTF_ENGINE_EXACT) otf_launch_exact(b, s);
    else if (engine == OTF_ENGINE_WINDOWED) {
        if (b.shared_bytes <= 0) return fail(OTF_EINVAL, "otf_run_batch: windowed engine needs shared_bytes");
        if (otf_launch_windowed(b, s) != 0) return fail(OTF_ECUDA, "otf_run_batch: shared memory request too large");
    }
    else return fail(OTF_EINVAL, "otf_run_batch: unknown engine");
    int rc = check_cuda("otf_run_batch");
    if (rc != OTF_OK || (b.engine_flags & OTF_BF_ENGINE_ONLY)) return rc;
    return otf_run_summary(batch, engine, stream);
}

int otf_run_summary(const otf_batch *batch, int32_t engine, void *stream) {
    if (!batch || batch->n_scenarios < 0) return fail(OTF_EINVAL, "otf_run_summary: bad batch");
    if (batch->n_scenarios == 0) return OTF_OK;
    if (otf_launch_summary(*batch, engine, (cudaStream_t)stream) != 0)
        return fail(OTF_ECUDA, "otf_run_summary: shared memory request too large");
    return check_cuda("otf_run_summary");
}

}  // extern "C"
