// otf_hostgen.cu -- HOST-side input generators of libotfgpu.so (include/otfgpu.h).
//
// The reference draws its per-run streams with numpy
// Generator(PCG64(SeedSequence(entropy))):
//   * arrival offsets  cumsum(exponential(1/rate, N))      SS([seed, 1])    orchestrator.py:265-268
//   * trace normals    standard_normal(n + 1) per client   SS([seed, 2, c]) orchestrator.py:254-263
//   * worker noise     normal(0, noise) per worker         SS([seed, w])    transcode.py:89-99
// and turns the normals into bandwidth samples with math.exp (glibc) and a
// CPython-3.12 compensated sum (netem.py:39-64,179-202).  These run here, on
// the host, with the same libm as numpy/CPython, and with all host threads:
// glibc's exp is what makes the trace values bit-exact, so this part stays on
// the CPU.  numpy's algorithms restated (numpy 2.3.5):
//   * SeedSequence + PCG64 (otf_rng.cuh, shared with the device);
//   * random_standard_normal / random_standard_exponential: 256-layer
//     ziggurats (numpy/random/src/distributions/distributions.c) over the
//     tables in otf_ziggurat.h;
//   * next_double = (next_uint64 >> 11) * 2^-53.
// Compiled with -ffp-contract=off: numpy's x86-64 baseline build does not fuse.
#include <math.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "otf_rng.cuh"
#include "otf_ziggurat.h"
#include "otfgpu.h"

int otf_fail(int code, const std::string &msg);

namespace otf {

// Generator.standard_normal (distributions.c random_standard_normal)
static double np_standard_normal(Pcg64 &g) {
    for (;;) {
        uint64_t r = pcg_next64(g);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 0x1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        double x = (double)rabs * zig::wi[idx];
        if (sign & 0x1) x = -x;
        if (rabs < zig::ki[idx]) return x;             // ~99.3% of draws
        if (idx == 0) {                                // tail beyond r (1 - U avoids log(0))
            for (;;) {
                double xx = -zig::nor_inv_r * log1p(-pcg_next_double(g));
                double yy = -log1p(-pcg_next_double(g));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 0x1) ? -(zig::nor_r + xx) : zig::nor_r + xx;
            }
        } else {
            if (((zig::fi[idx - 1] - zig::fi[idx]) * pcg_next_double(g) + zig::fi[idx]) < exp(-0.5 * x * x))
                return x;
        }
    }
}

// Generator.standard_exponential (distributions.c random_standard_exponential)
static double np_standard_exponential(Pcg64 &g) {
    for (;;) {
        uint64_t ri = pcg_next64(g);
        ri >>= 3;
        int idx = (int)(ri & 0xff);
        ri >>= 8;
        double x = (double)ri * zig::we[idx];
        if (ri < zig::ke[idx]) return x;               // ~98.9% of draws
        if (idx == 0) return zig::exp_r - log1p(-pcg_next_double(g));
        if ((zig::fe[idx - 1] - zig::fe[idx]) * pcg_next_double(g) + zig::fe[idx] < exp(-x)) return x;
    }
}

static void seed_stream(Pcg64 &g, const uint64_t *entropy, int n_entropy) {
    uint32_t words[64];
    int m = 0;
    for (int i = 0; i < n_entropy; i++) m = push_words(words, m, entropy[i]);
    pcg_seed(g, words, m);
}

// CPython >= 3.12 builtin sum() over floats: Neumaier-compensated.
double py_sum(const double *xs, int n) {
    double f = 0.0, c = 0.0;
    for (int i = 0; i < n; i++) {
        double x = xs[i];
        double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    }
    if (c != 0.0 && std::isfinite(c)) f += c;
    return f;
}

// synthetic_trace (netem.py:190-201) from its normals z[0..n], then
// BandwidthTrace._period_bits (netem.py:61-64).
static void trace_from_normals(const double *z, int32_t n, const double *starts, double period, double mu,
                               double sigma, double decay, double spread, double floor_bps, double cap_bps,
                               double *v, double *pbits, double *terms) {
    double x = mu + sigma * z[0];
    for (int32_t i = 0; i < n; i++) {
        double e = exp(x);                             // glibc exp == math.exp
        double bw = e > floor_bps ? e : floor_bps;
        bw = cap_bps < bw ? cap_bps : bw;
        v[i] = bw;
        x = mu + (x - mu) * decay + spread * z[i + 1];
    }
    for (int32_t i = 0; i < n; i++) {
        double end = (i + 1 < n) ? starts[i + 1] : period;
        terms[i] = v[i] * (end - starts[i]);
    }
    *pbits = py_sum(terms, n);
}

template <class F>
static void parallel_for(int64_t n, int n_threads, int64_t grain, F &&body) {
    int nt = (int)std::max<int64_t>(1, std::min<int64_t>(n_threads > 0 ? n_threads : 1, n / std::max<int64_t>(1, grain)));
    if (nt <= 1) { body((int64_t)0, n); return; }
    std::vector<std::thread> th;
    int64_t chunk = (n + nt - 1) / nt;
    for (int i = 0; i < nt; i++) {
        int64_t lo = i * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) th.emplace_back([&body, lo, hi] { body(lo, hi); });
    }
    for (auto &t : th) t.join();
}

}  // namespace otf

extern "C" {

int otf_np_draws(int32_t kind, const uint64_t *entropy, int32_t n_entropy, double loc, double scale, int64_t n,
                 double *out) {
    if (n < 0 || (n > 0 && !out) || n_entropy < 1 || n_entropy > 16 || !entropy)
        return otf_fail(OTF_EINVAL, "otf_np_draws: bad arguments");
    otf::Pcg64 g;
    otf::seed_stream(g, entropy, n_entropy);
    switch (kind) {
    case OTF_DRAW_STANDARD_NORMAL:
        for (int64_t i = 0; i < n; i++) out[i] = otf::np_standard_normal(g);
        break;
    case OTF_DRAW_NORMAL:                              // random_normal: loc + scale * z
        for (int64_t i = 0; i < n; i++) out[i] = loc + scale * otf::np_standard_normal(g);
        break;
    case OTF_DRAW_EXPONENTIAL:                         // random_exponential: scale * e
        for (int64_t i = 0; i < n; i++) out[i] = scale * otf::np_standard_exponential(g);
        break;
    case OTF_DRAW_STANDARD_EXPONENTIAL:
        for (int64_t i = 0; i < n; i++) out[i] = otf::np_standard_exponential(g);
        break;
    default:
        return otf_fail(OTF_EINVAL, "otf_np_draws: unknown kind");
    }
    return OTF_OK;
}

int otf_gen_arrivals(uint64_t seed, int64_t n, double scale, double *out) {
    if (n < 0 || (n > 0 && !out)) return otf_fail(OTF_EINVAL, "otf_gen_arrivals: bad arguments");
    uint64_t ent[2] = {seed, 1};
    otf::Pcg64 g;
    otf::seed_stream(g, ent, 2);
    double acc = 0.0;                                  // np.cumsum: sequential
    for (int64_t i = 0; i < n; i++) {
        acc += scale * otf::np_standard_exponential(g);
        out[i] = acc;
    }
    return OTF_OK;
}

int otf_gen_noise(uint64_t seed, int32_t n_workers, double noise, int64_t n, double *out, int32_t n_threads) {
    if (n_workers < 0 || n < 0 || (n_workers > 0 && n > 0 && !out))
        return otf_fail(OTF_EINVAL, "otf_gen_noise: bad arguments");
    otf::parallel_for(n_workers, n_threads, 1, [&](int64_t lo, int64_t hi) {
        for (int64_t w = lo; w < hi; w++) {
            uint64_t ent[2] = {seed, (uint64_t)w};
            otf::Pcg64 g;
            otf::seed_stream(g, ent, 2);
            double *o = out + w * n;
            for (int64_t i = 0; i < n; i++) o[i] = 0.0 + noise * otf::np_standard_normal(g);
        }
    });
    return OTF_OK;
}

int otf_gen_traces(uint64_t seed, int64_t n_traces, int32_t n_samples, const double *starts, double period,
                   double mu, double sigma, double decay, double spread, double floor_bps, double cap_bps,
                   double *values, double *pbits, int32_t n_threads) {
    if (n_traces < 0 || n_samples <= 0 || !starts || (n_traces > 0 && (!values || !pbits)))
        return otf_fail(OTF_EINVAL, "otf_gen_traces: bad arguments");
    otf::parallel_for(n_traces, n_threads, 16, [&](int64_t lo, int64_t hi) {
        std::vector<double> z((size_t)n_samples + 1), terms((size_t)n_samples);
        for (int64_t c = lo; c < hi; c++) {
            uint64_t ent[3] = {seed, 2, (uint64_t)c};
            otf::Pcg64 g;
            otf::seed_stream(g, ent, 3);
            for (int32_t i = 0; i <= n_samples; i++) z[(size_t)i] = otf::np_standard_normal(g);
            otf::trace_from_normals(z.data(), n_samples, starts, period, mu, sigma, decay, spread, floor_bps,
                                    cap_bps, values + c * (int64_t)n_samples, pbits + c, terms.data());
        }
    });
    return OTF_OK;
}

int otf_gen_traces_multi(int32_t n_jobs, const otf_trace_job *jobs, int32_t n_threads) {
    if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return otf_fail(OTF_EINVAL, "otf_gen_traces_multi: bad arguments");
    std::vector<int64_t> first((size_t)n_jobs + 1, 0);   // flattened (job, client) index space
    for (int32_t q = 0; q < n_jobs; q++) {
        const otf_trace_job &J = jobs[q];
        if (J.n_traces < 0 || J.n_samples <= 0 || !J.starts || (J.n_traces > 0 && (!J.values || !J.pbits)))
            return otf_fail(OTF_EINVAL, "otf_gen_traces_multi: bad job");
        first[(size_t)q + 1] = first[(size_t)q] + J.n_traces;
    }
    otf::parallel_for(first[(size_t)n_jobs], n_threads, 16, [&](int64_t lo, int64_t hi) {
        std::vector<double> z, terms;
        int32_t q = (int32_t)(std::upper_bound(first.begin(), first.end(), lo) - first.begin()) - 1;
        for (int64_t t = lo; t < hi; t++) {
            while (t >= first[(size_t)q + 1]) q++;
            const otf_trace_job &J = jobs[q];
            const int64_t c = t - first[(size_t)q];
            z.resize((size_t)J.n_samples + 1);
            terms.resize((size_t)J.n_samples);
            uint64_t ent[3] = {J.seed, 2, (uint64_t)c};
            otf::Pcg64 g;
            otf::seed_stream(g, ent, 3);
            for (int32_t i = 0; i <= J.n_samples; i++) z[(size_t)i] = otf::np_standard_normal(g);
            otf::trace_from_normals(z.data(), J.n_samples, J.starts, J.period, J.mu, J.sigma, J.decay, J.spread,
                                    J.floor_bps, J.cap_bps, J.values + c * (int64_t)J.n_samples, J.pbits + c,
                                    terms.data());
        }
    });
    return OTF_OK;
}

int otf_build_traces(int64_t n_traces, int32_t n_samples, const double *normals, const double *starts,
                     double period, double mu, double sigma, double decay, double spread,
                     double floor_bps, double cap_bps, double *values, double *pbits, int32_t n_threads) {
    if (n_traces < 0 || n_samples <= 0 || !normals || !starts || !values || !pbits)
        return otf_fail(OTF_EINVAL, "otf_build_traces: bad arguments");
    otf::parallel_for(n_traces, n_threads, 64, [&](int64_t lo, int64_t hi) {
        std::vector<double> terms((size_t)n_samples);
        for (int64_t t = lo; t < hi; t++)
            otf::trace_from_normals(normals + t * (int64_t)(n_samples + 1), n_samples, starts, period, mu, sigma,
                                    decay, spread, floor_bps, cap_bps, values + t * (int64_t)n_samples, pbits + t,
                                    terms.data());
    });
    return OTF_OK;
}

}  // extern "C"
