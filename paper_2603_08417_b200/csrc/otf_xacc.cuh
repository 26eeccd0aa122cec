// otf_xacc.cuh -- exact, order-independent sums of non-negative doubles.
//
// A fixed-point accumulator of XACC_LIMBS limbs, 32 payload bits each in a
// 64-bit word (bit 0 of limb 0 weighs 2^-128).  A double is split into at
// most three 32-bit chunks and added with integer (atomic) adds; the carries
// pile up in the upper halves of the words and are propagated once at the
// end, then the total is rounded to the nearest double (ties to even).  The
// result is the correctly rounded exact sum -- what Python's math.fsum
// returns -- whatever the order in which lanes, warps and scenarios add
// their terms, so device sums are bit-reproducible and checkable.
//
// Covered range: normal values in [2^-76, 2^64) (request latencies, startup
// delays).  Anything else sets XACC_INEXACT in the caller's flag word.
#pragma once
#include <stdint.h>

namespace otf {

constexpr int XACC_LIMBS = 8;
constexpr int XACC_BIAS = 128;                 // bit position of 2^0
constexpr uint32_t XACC_INEXACT = 0x2;         // == OTF_Q_INEXACT_SUM

// the (up to) three 32-bit chunks of v in limbs q, q+1, q+2; false when v is
// outside the covered range (v == 0 gives zero chunks)
__host__ __device__ __forceinline__ bool xacc_split(double v, int &q, uint32_t &c0, uint32_t &c1, uint32_t &c2) {
    c0 = c1 = c2 = 0;
    q = 0;
    if (v == 0.0) return true;
    uint64_t bits;
#ifdef __CUDA_ARCH__
    bits = (uint64_t)__double_as_longlong(v);
#else
    __builtin_memcpy(&bits, &v, 8);
#endif
    const int e = (int)((bits >> 52) & 0x7ff);
    if ((bits >> 63) || e == 0 || e == 0x7ff) return false;          // negative, subnormal, inf / nan
    const uint64_t m = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int p = e - 1075 + XACC_BIAS;                              // weight of m's lowest bit
    if (p < 0 || p + 85 > 32 * XACC_LIMBS - 32) return false;        // keep a limb of carry headroom
    q = p >> 5;
    const int r = p & 31;
    const unsigned __int128 x = (unsigned __int128)m << r;           // <= 85 bits
    c0 = (uint32_t)x;
    c1 = (uint32_t)(x >> 32);
    c2 = (uint32_t)(x >> 64);
    return true;
}

#ifdef __CUDACC__
// add v (any thread; limbs in shared or global memory)
__device__ __forceinline__ void xacc_add(unsigned long long *limb, double v, uint32_t *flags) {
    int q;
    uint32_t c0, c1, c2;
    if (!xacc_split(v, q, c0, c1, c2)) { atomicOr(flags, XACC_INEXACT); return; }
    if (c0) atomicAdd(limb + q, (unsigned long long)c0);
    if (c1) atomicAdd(limb + q + 1, (unsigned long long)c1);
    if (c2) atomicAdd(limb + q + 2, (unsigned long long)c2);
}
#endif

// carry-propagate a copy of the limbs and round to the nearest double
__host__ __device__ inline double xacc_round(const unsigned long long *limb_in) {
    uint64_t l[XACC_LIMBS];
    uint64_t carry = 0;
    for (int i = 0; i < XACC_LIMBS; i++) {
        const uint64_t v = (uint64_t)limb_in[i] + carry;             // < 2^64: carries are < 2^33
        l[i] = v & 0xffffffffull;
        carry = v >> 32;
    }
    int t = XACC_LIMBS - 1;
    while (t >= 0 && l[t] == 0) t--;
    if (t < 0) return 0.0;
    const unsigned __int128 x = ((unsigned __int128)l[t] << 64) | ((unsigned __int128)(t >= 1 ? l[t - 1] : 0) << 32) |
                                (unsigned __int128)(t >= 2 ? l[t - 2] : 0);
    bool sticky = false;
    for (int i = 0; i < t - 2; i++) sticky |= l[i] != 0;
    const int base = 32 * (t - 2) - XACC_BIAS;                       // weight exponent of x's bit 0
    int h = 64;                                                      // top set bit of x
    {
        uint64_t top = l[t];
        int lz = 0;
        while (!(top & 0x80000000ull)) { top <<= 1; lz++; }
        h = 64 + 31 - lz;
    }
    double m;
    int sh = 0;
    if (h <= 52) {
        m = (double)(uint64_t)x;                                     // exact, nothing below
    } else {
        sh = h - 52;
        uint64_t mm = (uint64_t)(x >> sh);
        const unsigned __int128 rem = x & (((unsigned __int128)1 << sh) - 1);
        const unsigned __int128 half = (unsigned __int128)1 << (sh - 1);
        if (rem > half || (rem == half && (sticky || (mm & 1)))) mm++;
        m = (double)mm;                                              // <= 2^53: exact
    }
    return ldexp(m, base + sh);
}

}  // namespace otf
