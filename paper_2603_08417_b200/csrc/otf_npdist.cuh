// otf_npdist.cuh -- numpy's Generator.standard_normal / standard_exponential,
// on host and device.
//
// numpy 2.3.5 numpy/random/src/distributions/distributions.c:
// random_standard_normal and random_standard_exponential are 256-layer
// ziggurats over next_uint64 (PCG64, otf_rng.cuh), with next_double =
// (next_uint64 >> 11) * 2^-53 in the wedge and tail tests.  Their libm calls
// (exp in the wedge test, log1p in the tail) go through otf_libm.cuh, the
// bit-exact restatement of the glibc the reference runs on, so the same code
// replays the reference's streams on the GPU (otf_gen.cu) and on the host
// (otf_hostgen.cu).  The rare branches (wedge ~0.7%, tail ~0.03% of normal
// draws) are kept out of line so the common path stays short.
#pragma once
#include <stdint.h>

#include "otf_libm.cuh"
#include "otf_rng.cuh"
#include "otf_ziggurat.h"

namespace otf {

struct ZigLayer { uint64_t k; double w, f; };

OTF_HD ZigLayer zig_nor(int i) {
#ifdef __CUDA_ARCH__
    const zig::Layer *L = &zig::nor_dev[i];
    return {__ldg((const unsigned long long *)&L->k), __ldg(&L->w), __ldg(&L->f)};
#else
    return {zig::ki[i], zig::wi[i], zig::fi[i]};
#endif
}

OTF_HD ZigLayer zig_exp(int i) {
#ifdef __CUDA_ARCH__
    const zig::Layer *L = &zig::exp_dev[i];
    return {__ldg((const unsigned long long *)&L->k), __ldg(&L->w), __ldg(&L->f)};
#else
    return {zig::ke[i], zig::we[i], zig::fe[i]};
#endif
}

#ifdef __CUDA_ARCH__
#define OTF_COLD __device__ __noinline__
#else
#define OTF_COLD static inline
#endif

// Tail beyond r (idx 0) or wedge test for one rejected normal draw: returns
// 1 and sets *out when the draw is accepted, 0 when the draw starts over.
OTF_COLD int np_normal_slow(Pcg64 &g, int idx, uint64_t rabs, double x, double *out) {
    if (idx == 0) {
        for (;;) {                                     // 1 - U avoids log(0)
            double xx = -zig::nor_inv_r * libm::log1p(-pcg_next_double(g));
            double yy = -libm::log1p(-pcg_next_double(g));
            if (yy + yy > xx * xx) {
                *out = ((rabs >> 8) & 0x1) ? -(zig::nor_r + xx) : zig::nor_r + xx;
                return 1;
            }
        }
    }
    const double f0 = zig_nor(idx - 1).f, f1 = zig_nor(idx).f;
    if (((f0 - f1) * pcg_next_double(g) + f1) < libm::exp(-0.5 * x * x)) { *out = x; return 1; }
    return 0;
}

// Generator.standard_normal (random_standard_normal)
OTF_HD double np_standard_normal(Pcg64 &g) {
    for (;;) {
        uint64_t r = pcg_next64(g);
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 0x1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        const ZigLayer L = zig_nor(idx);
        double x = (double)rabs * L.w;
        if (sign & 0x1) x = -x;
        if (rabs < L.k) return x;                      // ~99.3% of draws
        double out;
        if (np_normal_slow(g, idx, rabs, x, &out)) return out;
    }
}

OTF_COLD int np_exponential_slow(Pcg64 &g, int idx, double x, double *out) {
    if (idx == 0) { *out = zig::exp_r - libm::log1p(-pcg_next_double(g)); return 1; }
    const double f0 = zig_exp(idx - 1).f, f1 = zig_exp(idx).f;
    if ((f0 - f1) * pcg_next_double(g) + f1 < libm::exp(-x)) { *out = x; return 1; }
    return 0;
}

// Generator.standard_exponential (random_standard_exponential)
OTF_HD double np_standard_exponential(Pcg64 &g) {
    for (;;) {
        uint64_t ri = pcg_next64(g);
        ri >>= 3;
        const int idx = (int)(ri & 0xff);
        ri >>= 8;
        const ZigLayer L = zig_exp(idx);
        const double x = (double)ri * L.w;
        if (ri < L.k) return x;                        // ~98.9% of draws
        double out;
        if (np_exponential_slow(g, idx, x, &out)) return out;
    }
}

// CPython >= 3.12 builtin sum() over floats (Neumaier-compensated), one term at a time.
struct PySum {
    double f = 0.0, c = 0.0;
    OTF_HD void add(double x) {
        const double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else c += (x - t) + f;
        f = t;
    }
    OTF_HD double result() const { return (c != 0.0 && isfinite(c)) ? f + c : f; }
};

}  // namespace otf
