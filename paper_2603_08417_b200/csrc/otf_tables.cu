// otf_tables.cu -- request-generation tables built on the device.
//
// Segment sizes: Catalog.descriptor (content.py:204-218) derives each
// segment's jittered size from its own Generator(PCG64(SeedSequence([seed,
// sha256(seq)[:8], rank, index]))).  In the reference this is ~50% of the
// CPU time; here one thread per (sequence, rank, index)
// runs SeedSequence + PCG64 + one uniform draw, and the table is shared by
// every scenario with the same catalog.
#include <math.h>
#include <stdint.h>

#include "otf_model.cuh"
#include "otf_rng.cuh"
#include "otfgpu.h"

namespace otf {

__global__ void __launch_bounds__(256) sizes_kernel(const otf_size_table *tables, int64_t *i64_pool,
                                                    const double *f64_pool, const int32_t *i32_pool) {
    const otf_size_table t = tables[blockIdx.x];
    const int64_t n = (int64_t)t.n_seq * t.n_ranks * t.max_nseg;
    const int64_t *keys = i64_pool + t.off_keys;
    const int64_t *bitrates = i64_pool + t.off_bitrates;
    const double *seqdur = f64_pool + t.off_seqdur;
    const double *segdur = f64_pool + t.off_segdur;
    const int32_t *counts = i32_pool + t.off_segcount;
    int64_t *out = i64_pool + t.off_out;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
        int32_t index = (int32_t)(e % t.max_nseg);
        int32_t rank = (int32_t)((e / t.max_nseg) % t.n_ranks) + 1;
        int32_t seq = (int32_t)(e / ((int64_t)t.max_nseg * t.n_ranks));
        if (index >= counts[seq]) { out[e] = 0; continue; }
        double duration = seg_duration(seqdur[seq], segdur[seq], index);
        double base = ((double)bitrates[rank - 1] * duration) / 8.0;
        uint32_t ent[12];
        int m = 0;
        m = push_words(ent, m, t.seed);
        m = push_words(ent, m, (uint64_t)keys[seq]);
        m = push_words(ent, m, (uint64_t)rank);
        m = push_words(ent, m, (uint64_t)index);
        Pcg64 g;
        pcg_seed(g, ent, m);
        double j = t.size_jitter;
        double u = -j + (j - -j) * pcg_next_double(g);     // Generator.uniform(-j, j)
        double v = rint(base * (1.0 + u));                 // round(): half-to-even
        int64_t size = (int64_t)v;
        out[e] = size > 1 ? size : 1;                      // max(1, ...)
    }
}

}  // namespace otf

int otf_launch_sizes(const otf_size_table *tables_dev, int32_t n_tables, int64_t *i64_pool,
                     const double *f64_pool, const int32_t *i32_pool, cudaStream_t stream) {
    if (n_tables <= 0) return 0;
    otf::sizes_kernel<<<n_tables, 256, 0, stream>>>(tables_dev, i64_pool, f64_pool, i32_pool);
    return 0;
}
