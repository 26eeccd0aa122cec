// otf_hostgen.cu -- HOST-side input generators of libotfgpu.so (include/otfgpu.h).
//
// The reference draws its per-run streams with numpy
// Generator(PCG64(SeedSequence(entropy))):
//   * arrival offsets  cumsum(exponential(1/rate, N))      SS([seed, 1])    orchestrator.py:265-268
//   * trace normals    standard_normal(n + 1) per client   SS([seed, 2, c]) orchestrator.py:254-263
//   * worker noise     normal(0, noise) per worker         SS([seed, w])    transcode.py:89-99
// and turns the normals into bandwidth samples with math.exp (glibc) and a
// CPython-3.12 compensated sum (netem.py:39-64,179-202).  These run here, on
// the host, with all host threads.  The product path generates the same
// tables on the device (otf_gen.cu); these host generators are the C-ABI
// replicas the tests pin against numpy, sharing every line of arithmetic with
// the device through otf_npdist.cuh (numpy 2.3.5's ziggurats over
// SeedSequence + PCG64) and otf_libm.cuh (glibc's exp / log1p).
// Compiled with -ffp-contract=off: numpy's x86-64 baseline build does not fuse.
#include <math.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "otf_npdist.cuh"
#include "otfgpu.h"

int otf_fail(int code, const std::string &msg);

namespace otf {

static void seed_stream(Pcg64 &g, const uint64_t *entropy, int n_entropy) {
    uint32_t words[64];
    int m = 0;
    for (int i = 0; i < n_entropy; i++) m = push_words(words, m, entropy[i]);
    pcg_seed(g, words, m);
}

// CPython >= 3.12 builtin sum() over floats: Neumaier-compensated.
double py_sum(const double *xs, int n) {
    PySum s;
    for (int i = 0; i < n; i++) s.add(xs[i]);
    return s.result();
}

// synthetic_trace (netem.py:190-201) from its normals z[0..n], then
// BandwidthTrace._period_bits (netem.py:61-64).
static void trace_from_normals(const double *z, int32_t n, const double *starts, double period, double mu,
                               double sigma, double decay, double spread, double floor_bps, double cap_bps,
                               double *v, double *pbits, double *terms) {
    double x = mu + sigma * z[0];
    for (int32_t i = 0; i < n; i++) {
        double e = libm::exp(x);                       // == math.exp (glibc, otf_libm.cuh)
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
