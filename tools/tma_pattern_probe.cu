// HBM read rate of the weight-streaming access pattern (tool, not product).
// Each CTA streams `tiles` 128-row weight tiles of a [N][K] bf16 matrix
// (K = 4096, the Mixtral-8x7B d) along K, one 64-column k-block per stage:
//   tma2d   : 2D TMA box 128 rows x 64 cols (128 B per row, rows 8 KB apart),
//             the layout kl_gemm_bf16's streaming kernel reads today
//   tiled   : the same bytes pre-tiled so each (row tile, k-block) is one
//             contiguous 16 KB block, loaded with one 1D cp.async.bulk
// Grid = 112 (the whole-tile SwiGLU GEMM) or 148 CTAs; `stages` deep ring;
// one consumer thread just releases slots. Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -Ipaper_2502_06888_b200/csrc/kernels -Iinclude -o tools/tma_pattern_probe tools/tma_pattern_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "tma_host.cuh"

using namespace kl;

constexpr int kRows = 128, kBK = 64, kTile = kRows * kBK * 2;  // 16 KB

__global__ void stream_ring(const __grid_constant__ CUtensorMap map, const char* __restrict__ tiled, int K,
                            int tiles_per_cta, int nt_stage, int stages, int mode) {
    extern __shared__ __align__(1024) char sm[];
    const int stage_bytes = nt_stage * kTile;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * stage_bytes);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int KB = K / kBK;
    const int groups = tiles_per_cta / nt_stage;  // tile groups walked one after another
    const int total = groups * KB;
    if (threadIdx.x == 0) {
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            if (it >= stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            const int g = it / KB, kb = it % KB;
            for (int j = 0; j < nt_stage; ++j) {
                const int tile = (blockIdx.x * tiles_per_cta) + g * nt_stage + j;
                char* dst = sm + static_cast<size_t>(s) * stage_bytes + j * kTile;
                if (mode == 0)
                    tma_load_2d(dst, &map, &full[s], kb * kBK, tile * kRows);
                else
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(dst)),
                        "l"(tiled + (static_cast<int64_t>(tile) * KB + kb) * kTile), "r"(kTile),
                        "r"(smem_u32(&full[s]))
                        : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            mbar_wait(&full[s], (it / stages) & 1);
            mbar_arrive(&empty[s]);
        }
    }
}

int main() {
    const int K = 4096;
    const int64_t N = 28672 * 4;  // 4 SwiGLU weight sets (940 MB) so launches rotate past L2
    const int64_t bytes = N * K * 2;
    char* buf = nullptr;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{");
    const char* sep = "";
    struct Cfg {
        int ctas, tiles, nt, stages, mode;
    };
    // Per launch: one 235 MB weight set (224 row tiles of 128 rows).
    const Cfg cfgs[] = {{112, 2, 2, 4, 0}, {112, 2, 2, 4, 1}, {112, 2, 2, 6, 1}, {112, 2, 1, 8, 0},
                        {112, 2, 1, 8, 1}, {224, 1, 1, 6, 0}, {224, 1, 1, 6, 1}, {112, 2, 2, 3, 0}};
    for (const Cfg& c : cfgs) {
        CUtensorMap maps[4];
        for (int r = 0; r < 4; ++r)
            if (make_map(&maps[r], buf + r * (bytes / 4), N / 4, K, kRows)) {
                printf("\"err\": \"map\"}\n");
                return 1;
            }
        const int smem = c.stages * c.nt * kTile + 1024;
        cudaFuncSetAttribute(stream_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int r = 0;
        auto launch = [&] {
            const int q = r++ % 4;
            stream_ring<<<c.ctas, 64, smem>>>(maps[q], buf + q * (bytes / 4), K, c.tiles, c.nt, c.stages, c.mode);
        };
        for (int w = 0; w < 4; ++w) launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        const int iters = 16;
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double per = static_cast<double>(c.ctas) * c.tiles * kTile * (K / kBK);
        printf("%s\"%s_ctas%d_nt%d_s%d\": {\"us\": %.1f, \"GBs\": %.0f}", sep, c.mode ? "tiled" : "tma2d", c.ctas, c.nt,
               c.stages, ms * 1e3 / iters, per * iters / (ms * 1e-3) / 1e9);
        sep = ", ";
    }
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
