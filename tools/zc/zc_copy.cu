// Probe: SM-driven host->device copy (zero-copy loads from pinned host
// memory through UVA, 16-byte vector stores to HBM). Used by
// tools/op_latency_probe.py to test whether a copy issued by SMs instead of
// the copy engine disturbs a concurrent HBM-streaming kernel.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void zc_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x); i < n16; i += stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t j = i + static_cast<int64_t>(u) * gridDim.x * blockDim.x;
            if (j < n16) v[u] = __ldcs(src + j);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t j = i + static_cast<int64_t>(u) * gridDim.x * blockDim.x;
            if (j < n16) __stcs(dst + j, v[u]);
        }
    }
}

extern "C" int zc_copy(void* dst, const void* src, int64_t bytes, int ctas, int threads, cudaStream_t st) {
    zc_copy_kernel<<<ctas, threads, 0, st>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), bytes / 16);
    return static_cast<int>(cudaGetLastError());
}
