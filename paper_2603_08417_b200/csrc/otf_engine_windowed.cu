// placeholder: windowed engine (next milestone) -- routes to the exact engine.
#include <cuda_runtime.h>
#include <stdint.h>
#include "otfgpu.h"
#include "otf_state.cuh"
int otf_launch_exact(const otf_batch &b, cudaStream_t stream);
int64_t otf_windowed_scratch_bytes(int32_t n_clients, int32_t n_workers, int64_t n_desc) {
    return otf::exact_layout(n_clients, n_workers, n_desc).total;
}
int otf_launch_windowed(const otf_batch &b, cudaStream_t stream) { return otf_launch_exact(b, stream); }
