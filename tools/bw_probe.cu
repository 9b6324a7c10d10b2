// HBM read-bandwidth probe (tool, not product): plain LDG.128 streams and
// 1D bulk-copy (cp.async.bulk) rings of several depths / sizes, timed with
// CUDA events over a buffer much larger than L2. Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void ldg_sum(const uint4* __restrict__ p, int64_t n, uint32_t* out) {
    uint32_t acc = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n; i += stride) {
        const uint4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// One CTA per SM; a ring of `stages` slots of `chunk` bytes; one thread
// issues 1D bulk copies of `piece` bytes; consumers just release.
__global__ void bulk_ring(const char* __restrict__ src, int64_t bytes, int chunk, int piece, int stages) {
    extern __shared__ __align__(128) char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * chunk);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int64_t n_chunks = bytes / chunk;
    const int64_t c0 = blockIdx.x * n_chunks / gridDim.x, c1 = (blockIdx.x + 1) * n_chunks / gridDim.x;
    if (threadIdx.x == 0) {
        int64_t it = 0;
        for (int64_t c = c0; c < c1; ++c, ++it) {
            const int s = static_cast<int>(it % stages);
            if (it >= stages) {
                const uint32_t par = static_cast<uint32_t>((it / stages + 1) & 1);
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                                 : "=r"(ok) : "r"(su32(&empty[s])), "r"(par) : "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
            for (int o = 0; o < chunk; o += piece)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su32(sm + static_cast<size_t>(s) * chunk + o)),
                             "l"(src + c * chunk + o), "r"(piece), "r"(su32(&full[s]))
                             : "memory");
        }
    } else if (threadIdx.x == 32) {
        int64_t it = 0;
        for (int64_t c = c0; c < c1; ++c, ++it) {
            const int s = static_cast<int>(it % stages);
            const uint32_t par = static_cast<uint32_t>((it / stages) & 1);
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(su32(&full[s])), "r"(par) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
    }
}

int main() {
    const int64_t bytes = 2LL << 30;  // 2 GiB >> L2
    char* buf = nullptr;
    uint32_t* out = nullptr;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](auto&& launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return bytes * 5 / (ms * 1e-3) / 1e9;
    };
    printf("{\"sms\": %d", sms);
    for (int bpsm : {4, 8, 16}) {
        const double gbs = time([&] { ldg_sum<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out); });
        printf(", \"ldg_%dx256\": %.0f", bpsm, gbs);
    }
    struct Cfg {
        int chunk, piece, stages, ctas_per_sm;
    };
    for (Cfg c : std::vector<Cfg>{{65536, 65536, 3, 1}, {65536, 2048, 3, 1}, {32768, 32768, 6, 1}, {16384, 16384, 12, 1},
                                  {65536, 65536, 2, 1}, {32768, 32768, 3, 2}, {16384, 16384, 4, 4}, {8192, 8192, 8, 2}}) {
        const size_t smem = static_cast<size_t>(c.chunk) * c.stages + 16 * c.stages;
        cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        const double gbs = time([&] { bulk_ring<<<sms * c.ctas_per_sm, 64, smem>>>(buf, bytes, c.chunk, c.piece, c.stages); });
        printf(", \"bulk_c%d_p%d_s%d_x%d\": %.0f", c.chunk, c.piece, c.stages, c.ctas_per_sm, gbs);
    }
    // Fewer CTAs than SMs (the whole-tile SwiGLU GEMM runs 112): can each SM
    // pull more than its 1/148 share?
    for (int ctas : {112, 128}) {
        const size_t smem = static_cast<size_t>(65536) * 3 + 48;
        cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        const double gbs = time([&] { bulk_ring<<<ctas, 64, smem>>>(buf, bytes, 65536, 65536, 3); });
        printf(", \"bulk_c65536_s3_ctas%d\": %.0f", ctas, gbs);
    }
    // Short launches (68 MB, the decode-attention size) rotating over 4
    // buffers so L2 (126 MB) never holds the next launch's bytes.
    {
        const int64_t small = 68LL << 20;
        for (Cfg c : std::vector<Cfg>{{65536, 65536, 3, 1}, {32768, 32768, 6, 1}, {32768, 32768, 3, 2}}) {
            const size_t smem = static_cast<size_t>(c.chunk) * c.stages + 16 * c.stages;
            cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            int r = 0;
            auto launch = [&] { bulk_ring<<<sms * c.ctas_per_sm, 64, smem>>>(buf + (r++ % 4) * small, small, c.chunk, c.piece, c.stages); };
            for (int w = 0; w < 8; ++w) launch();
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int i = 0; i < 40; ++i) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf(", \"short68MB_c%d_s%d_x%d_us\": %.2f", c.chunk, c.stages, c.ctas_per_sm, ms * 1e3 / 40);
        }
    }
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
