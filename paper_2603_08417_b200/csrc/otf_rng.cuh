// otf_rng.cuh -- numpy's SeedSequence + PCG64 stream, on the device.
//
// The reference derives every stream from numpy
// Generator(PCG64(SeedSequence([...]))) (content.py:165-167 segment sizes,
// orchestrator.py:340-342 sequence picks).  These are the integer algorithms
// of numpy 2.3.5 (bit_generator.pyx SeedSequence.mix_entropy/generate_state,
// pcg64.h pcg_setseq_128_xsl_rr_64), reproduced so that sizes and picks are
// generated on the GPU instead of being shipped as tables.
#pragma once
#include <stdint.h>

#ifndef OTF_HD
#define OTF_HD __host__ __device__ __forceinline__
#endif

namespace otf {

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
    uint32_t has_uint32, uinteger;
};

OTF_HD u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// numpy _int_to_uint32_array: little-endian 32-bit words, 0 -> [0].
OTF_HD int push_words(uint32_t *w, int n, uint64_t v) {
    if (v == 0) { w[n++] = 0; return n; }
    while (v) { w[n++] = (uint32_t)(v & 0xffffffffu); v >>= 32; }
    return n;
}

// SeedSequence(entropy words).generate_state(4, uint64) -> PCG64.__init__.
OTF_HD void pcg_seed(Pcg64 &g, const uint32_t *ent, int m) {
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
    auto hashmix = [&](uint32_t v) -> uint32_t {
        v ^= hc; hc *= 0x931e8875u; v *= hc; v ^= v >> 16; return v;
    };
    auto mix = [](uint32_t x, uint32_t y) -> uint32_t {
        uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y; r ^= r >> 16; return r;
    };
    // loops kept rolled: this runs once per stream and code size matters more
#pragma unroll 1
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < m ? ent[i] : 0u);
#pragma unroll 1
    for (int s = 0; s < 4; s++)
#pragma unroll 1
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
#pragma unroll 1
    for (int s = 4; s < m; s++)
#pragma unroll 1
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(ent[s]));
    uint32_t st[8];
    uint32_t hb = 0x8b51f9ddu;
#pragma unroll 1
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb; hb *= 0x58f38dedu; v *= hb; v ^= v >> 16;
        st[i] = v;
    }
    uint64_t v0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    uint64_t v1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
    uint64_t v2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
    uint64_t v3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
    u128 seed = ((u128)v0 << 64) | v1;
    u128 inc = ((u128)v2 << 64) | v3;
    g.inc = (inc << 1) | 1u;
    g.state = g.inc;                       // 0 * mult + inc
    g.state += seed;
    g.state = g.state * pcg_mult() + g.inc;
    g.has_uint32 = 0;
    g.uinteger = 0;
}

OTF_HD uint64_t pcg_next64(Pcg64 &g) {
    g.state = g.state * pcg_mult() + g.inc;
    uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

OTF_HD uint32_t pcg_next32(Pcg64 &g) {
    if (g.has_uint32) { g.has_uint32 = 0; return g.uinteger; }
    uint64_t n = pcg_next64(g);
    g.has_uint32 = 1;
    g.uinteger = (uint32_t)(n >> 32);
    return (uint32_t)n;
}

// Generator.random(): (next_uint64 >> 11) * 2^-53
OTF_HD double pcg_next_double(Pcg64 &g) {
    return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.integers(n), 1 <= n <= 2^32: numpy's buffered bounded Lemire (32-bit).
OTF_HD int32_t pcg_integers(Pcg64 &g, uint32_t n) {
    uint32_t rng = n - 1u;
    if (rng == 0) return 0;
    if (rng == 0xffffffffu) return (int32_t)pcg_next32(g);
    uint32_t r1 = rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(g) * r1;
    uint32_t left = (uint32_t)m;
    if (left < r1) {
        uint32_t thr = (0u - r1) % r1;
        while (left < thr) { m = (uint64_t)pcg_next32(g) * r1; left = (uint32_t)m; }
    }
    return (int32_t)(m >> 32);
}

}  // namespace otf
