// otf_libm.cuh -- glibc's exp() and log1p(), bit-for-bit, on host and device.
//
// The reference's streams pass through libm: bandwidth = math.exp(x)
// (netem.py:198), and numpy's ziggurats call exp() in the rejection test and
// log1p() in the tail (distributions.c random_standard_normal /
// random_standard_exponential).  CUDA's exp/log1p differ from glibc's in the
// last place, so the device generators use this restatement of the code the
// reference actually runs: glibc 2.39 on x86-64, whose ifunc selects the
// FMA builds (__exp_fma, __log1p_fma) on every AVX2+FMA host.  Every fused
// multiply-add below is one the compiler emitted in those builds (read from
// their disassembly); every other operation is a separately rounded one, so
// the file must be compiled without contraction (--fmad=false,
// -ffp-contract=off) -- the Makefile does.
//
// exp:   sysdeps/ieee754/dbl-64/e_exp.c (ARM optimized-routines exp, N = 128
//        table, degree-5 polynomial) incl. its specialcase() for |x| > 512;
// log1p: sysdeps/ieee754/dbl-64/s_log1p.c (fdlibm, R1..R4 split polynomial).
// The constants are in otf_libm_tab.h (tools/gen_libm_tables.py, checked
// against the installed libm).  tests/test_host.py and tests/test_gpu_gen.py
// compare both functions with the host libm on >= 1e7 / 1e8 arguments.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "otf_libm_tab.h"

#ifndef OTF_HD
#define OTF_HD __host__ __device__ __forceinline__
#endif

namespace otf { namespace libm {

OTF_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return ::fma(a, b, c);
#endif
}

OTF_HD uint64_t as_u64(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}

OTF_HD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x; memcpy(&x, &u, 8); return x;
#endif
}

OTF_HD uint64_t exp_tab(int i) {
#ifdef __CUDA_ARCH__
    return __ldg((const unsigned long long *)&exp_tab_dev[i]);
#else
    return exp_tab_host[i];
#endif
}

// e_exp.c specialcase(): 2^(k/N) * (1 + tmp) when the exponent of scale over/underflows
OTF_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {                   // k > 0
        sbits -= 1009ull << 52;
        double scale = as_f64(sbits);
        return fma_(scale, tmp, scale) * 0x1p1009;
    }
    sbits += 1022ull << 52;                            // k < 0: subnormal care
    double scale = as_f64(sbits);
    double st = scale * tmp;
    double y = scale + st;
    if (y < 1.0) {
        double hi = 1.0 + y;
        double lo = (scale - y) + st;
        lo = ((1.0 - hi) + y) + lo;
        y = (hi + lo) - 1.0;
        if (y == 0.0) y = 0.0;                         // no -0.0
    }
    return y * 0x1p-1022;
}

// glibc exp (the __exp_fma build)
OTF_HD double exp(double x) {
    uint64_t ux = as_u64(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x3fu) {                    // |x| < 2^-54 or |x| >= 512 (or inf/nan)
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;
        if (abstop >= 0x409u) {                        // |x| >= 1024
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (ux >> 63) ? 0.0 : as_f64(0x7ff0000000000000ull);
        }
        abstop = 0;                                    // large |x|: specialcase below
    }
    double kd = fma_(x, invln2N, shift);               // z + shift, fused
    uint64_t ki = as_u64(kd);
    kd -= shift;
    double r = fma_(kd, negln2hiN, x);
    r = fma_(kd, negln2loN, r);
    uint64_t idx = 2 * (ki % 128);
    uint64_t top = ki << 45;
    double tail = as_f64(exp_tab((int)idx));
    uint64_t sbits = exp_tab((int)idx + 1) + top;
    double p23 = fma_(r, C3, C2);
    double t0 = r + tail;
    double r2 = r * r;
    double p45 = fma_(r, C5, C4);
    double t1 = fma_(p23, r2, t0);
    double r4 = r2 * r2;
    double tmp = fma_(r4, p45, t1);
    if (abstop == 0) return exp_special(tmp, sbits, ki);
    double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
}

// glibc log1p (the __log1p_fma build of fdlibm's s_log1p.c)
OTF_HD double log1p(double x) {
    const uint64_t ux = as_u64(x);
    const int32_t hx = (int32_t)(ux >> 32);
    const int32_t ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    double f = 0.0, c = 0.0;
    if (hx < 0x3fda827a) {                             // x < 0.41422
        if (ax >= 0x3ff00000) {                        // x <= -1
            if (x == -1.0) return -as_f64(0x7ff0000000000000ull);
            return as_f64(0x7ff8000000000000ull);
        }
        if (ax < 0x3e200000) {                         // |x| < 2^-29
            if (ax < 0x3c900000) return x;
            return fma_(-(x * x), 0.5, x);
        }
        if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) { k = 0; f = x; hu = 1; }   // -0.2929 < x < 0.41422
                                                       // (hx > 0 || hx <= 0xbfd2bec3, as the build compares it)
    } else if (hx >= 0x7ff00000) {
        return x + x;
    }
    if (k != 0) {
        double u;
        if (hx < 0x43400000) {
            u = 1.0 + x;
            hu = (int32_t)(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
            c /= u;
        } else {
            u = x;
            hu = (int32_t)(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        const uint64_t lo = as_u64(u) & 0xffffffffull;
        if (hu < 0x6a09e) {
            u = as_f64(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo);
        } else {
            k += 1;
            u = as_f64(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo);
            hu = (0x00100000 - hu) >> 2;
        }
        f = u - 1.0;
    }
    const double hfsq = (f * 0.5) * f;
    if (hu == 0) {                                     // |f| < 2^-20 (only on the k != 0 path)
        const double dk = (double)k;
        if (f == 0.0) return k == 0 ? 0.0 : fma_(dk, ln2_hi, fma_(dk, ln2_lo, c));
        const double R = fma_(-f, two3, 1.0) * hfsq;
        if (k == 0) return f - R;
        return fma_(dk, ln2_hi, -((R - fma_(dk, ln2_lo, c)) - f));
    }
    const double s = f / (2.0 + f);
    const double z = s * s;
    const double R2 = fma_(z, Lp3, Lp2);
    const double R3 = fma_(z, Lp5, Lp4);
    const double R4 = fma_(z, Lp7, Lp6);
    const double z2 = z * z;
    const double z4 = z2 * z2;
    const double z6 = z2 * z4;
    double R = fma_(z, Lp1, z2 * R2);
    R = fma_(z4, R3, R);
    R = fma_(z6, R4, R);
    const double shr = (R + hfsq) * s;
    if (k == 0) return f - (hfsq - shr);
    const double dk = (double)k;
    return fma_(dk, ln2_hi, -(((hfsq - (fma_(dk, ln2_lo, c) + shr)) - f)));
}

}}  // namespace otf::libm
