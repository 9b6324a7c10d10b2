// SPDX-License-Identifier: Apache-2.0
// K5: bf16 GEMM / grouped expert FFN on 5th-gen tensor cores (sm_100a).
//
// One CTA computes one 128 x BN output tile:
//   warp 0   : TMA producer  (A and B tiles, 128B swizzle, STAGES-deep ring)
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5: epilogue (tcgen05.ld TMEM -> registers -> bf16 global stores);
//              warp w owns TMEM lanes 32*(w%4) .. +31 (= tile rows).
// Pipelines: smem full/empty mbarriers between TMA and MMA, one accumulator
// barrier between MMA (tcgen05.commit) and the epilogue.
//
// Used for the expert FFN (compute_expert, reference schedule.cpp:355-372:
// the reference only prices it at token_count * t_c_e_per_token,
// simulator.cpp:17) and for the attention projections (compute_attention).
// In decode (M <= a few hundred rows per expert) the kernel is HBM-bound on
// the weight stream: algorithmic bytes = 3*d*f*2 per expert.
#include <cuda.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"

namespace kl {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle span
constexpr int kThreads = 192;
constexpr int kSmemBudget = 200 * 1024;

enum Epilogue { kStore = 0, kResidual = 1, kSwiGLU = 2 };

template <int BN>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (kSmemBudget / kStageBytes) < 8 ? (kSmemBudget / kStageBytes) : 8;
    static constexpr int kTmemCols = BN;  // fp32 accumulator columns (power of two >= 32)
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  int a_row0, int M, int K, int b_half_rows, uint16_t* __restrict__ c, int ldc,
                  const uint16_t* __restrict__ r) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* acc_ready = empty + C::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n_tile = blockIdx.x;
    const int m_tile = blockIdx.y;
    const int num_kb = K / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_ready, 1);
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const int a_row = a_row0 + m_tile * BM;
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % C::kStages;
                const uint32_t phase = (kb / C::kStages) & 1;
                mbar_wait(&empty[s], phase ^ 1);
                uint8_t* sa = smem + s * C::kStageBytes;
                uint8_t* sb = sa + C::kABytes;
                mbar_arrive_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(sa, &tmap_a, &full[s], kb * BK, a_row);
                if constexpr (EPI == kSwiGLU) {
                    // [W1 rows | W3 rows] of this output column block, stacked along N.
                    tma_load_2d(sb, &tmap_b, &full[s], kb * BK, n_tile * (BN / 2));
                    tma_load_2d(sb + (BN / 2) * BK * 2, &tmap_b, &full[s], kb * BK,
                                b_half_rows + n_tile * (BN / 2));
                } else {
                    tma_load_2d(sb, &tmap_b, &full[s], kb * BK, n_tile * BN);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % C::kStages;
                const uint32_t phase = (kb / C::kStages) & 1;
                mbar_wait(&full[s], phase);
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + s * C::kStageBytes);
                const uint32_t sb = sa + C::kABytes;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // UMMA_K = 16 bf16 = 32 bytes along the swizzled row.
                    tc_mma_bf16(tmem_base, sw128_kmajor_desc(sa + k * 32), sw128_kmajor_desc(sb + k * 32), idesc,
                                (kb | k) != 0);
                }
                tc_commit(&empty[s]);  // smem stage reusable once these MMAs retire
            }
            tc_commit(acc_ready);  // accumulator complete
        }
        __syncwarp();
    } else {
        // Epilogue: 4 warps x 32 lanes = 128 tile rows.
        mbar_wait(acc_ready, 0);
        tc_fence_after();
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        const int row = m_tile * BM + row_in_tile;
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
        const bool live = row < M;
        if constexpr (EPI == kSwiGLU) {
            constexpr int HALF = BN / 2;
            uint16_t* out = c + static_cast<int64_t>(row) * ldc + n_tile * HALF;
#pragma unroll 1
            for (int col = 0; col < HALF; col += 16) {
                float g[16], u[16];
                tmem_ld16(lane_addr + col, g);
                tmem_ld16(lane_addr + HALF + col, u);
                if (live) {
                    uint32_t packed[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float a0 = g[2 * i] / (1.0f + expf(-g[2 * i])) * u[2 * i];
                        const float a1 = g[2 * i + 1] / (1.0f + expf(-g[2 * i + 1])) * u[2 * i + 1];
                        packed[i] = pack2(a0, a1);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(out + col);
                    dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
                    dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
                }
            }
        } else {
            uint16_t* out = c + static_cast<int64_t>(row) * ldc + n_tile * BN;
            const uint16_t* res = EPI == kResidual ? r + static_cast<int64_t>(row) * ldc + n_tile * BN : nullptr;
#pragma unroll 1
            for (int col = 0; col < BN; col += 16) {
                float v[16];
                tmem_ld16(lane_addr + col, v);
                if (live) {
                    if constexpr (EPI == kResidual) {
                        const uint4* rp = reinterpret_cast<const uint4*>(res + col);
                        const uint4 r0 = rp[0], r1 = rp[1];
                        const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            v[2 * i] += bf2f(static_cast<uint16_t>(rw[i] & 0xffffu));
                            v[2 * i + 1] += bf2f(static_cast<uint16_t>(rw[i] >> 16));
                        }
                    }
                    uint32_t packed[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) packed[i] = pack2(v[2 * i], v[2 * i + 1]);
                    uint4* dst = reinterpret_cast<uint4*>(out + col);
                    dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
                    dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::kTmemCols);
    }
}

// ------------------------------------------------------------ host side ----

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// Row-major bf16 matrix [rows, cols] viewed by TMA in boxes of [box_rows, 64].
int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeFn enc = encoder();
    if (enc == nullptr) return KL_ENODEV;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : KL_EINVAL;
}

template <int BN, int EPI>
int launch(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int64_t b_rows,
           int n_tiles, int b_half_rows, uint16_t* c, int ldc, const uint16_t* r, cudaStream_t stream) {
    using C = Cfg<BN>;
    CUtensorMap ma, mb;
    int rc = make_map(&ma, a, a_rows, K, BM);
    if (rc) return rc;
    rc = make_map(&mb, b, b_rows, K, EPI == kSwiGLU ? BN / 2 : BN);
    if (rc) return rc;
    static bool configured = false;  // per template instance
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes));
        configured = true;
    }
    const dim3 grid(n_tiles, (M + BM - 1) / BM);
    gemm_bf16_tcgen05<BN, EPI><<<grid, kThreads, C::kSmemBytes, stream>>>(
        ma, mb, static_cast<int>(row_offset), M, K, b_half_rows, c, ldc, r);
    return check_launch();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace kl

extern "C" int kl_gemm_bf16(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                            const uint16_t* b, int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue,
                            cudaStream_t stream) {
    using namespace kl;
    if (M < 0 || K <= 0 || N <= 0 || a == nullptr || b == nullptr || c == nullptr) return KL_EINVAL;
    if (M == 0) return KL_OK;
    if (K % BK != 0 || N % 64 != 0 || !aligned16(a) || !aligned16(b) || !aligned16(c) || ldc % 8 != 0)
        return KL_EINVAL;
    if (row_offset < 0 || row_offset + M > a_rows || row_offset > INT32_MAX) return KL_EINVAL;
    const int m_tiles = (M + BM - 1) / BM;
    switch (epilogue) {
        case kStore:
        case kResidual: {
            if (epilogue == kResidual && (r == nullptr || !aligned16(r))) return KL_EINVAL;
            // Narrow tiles when the grid would leave SMs idle (decode shapes are
            // weight-stream bound: more CTAs = more concurrent HBM streams).
            const bool narrow = (N / 128) * m_tiles < 148;
            if (epilogue == kStore)
                return narrow ? launch<64, kStore>(a, a_rows, row_offset, M, K, b, N, N / 64, 0, c, ldc, r, stream)
                              : launch<128, kStore>(a, a_rows, row_offset, M, K, b, N, N / 128, 0, c, ldc, r, stream);
            return narrow ? launch<64, kResidual>(a, a_rows, row_offset, M, K, b, N, N / 64, 0, c, ldc, r, stream)
                          : launch<128, kResidual>(a, a_rows, row_offset, M, K, b, N, N / 128, 0, c, ldc, r, stream);
        }
        case kSwiGLU: {
            if (N % 256 != 0) return KL_EINVAL;
            const int half = N / 2;  // b rows: [W1 (half) ; W3 (half)]
            const bool narrow = (N / 256) * m_tiles < 148;
            return narrow ? launch<128, kSwiGLU>(a, a_rows, row_offset, M, K, b, N, N / 128, half, c, ldc, r, stream)
                          : launch<256, kSwiGLU>(a, a_rows, row_offset, M, K, b, N, N / 256, half, c, ldc, r, stream);
        }
        default: return KL_EINVAL;
    }
}

extern "C" int kl_expert_ffn(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d, int f,
                             const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch, uint16_t* y,
                             cudaStream_t stream) {
    if (M == 0) return KL_OK;
    if (y == nullptr || h_scratch == nullptr) return KL_EINVAL;
    int rc = kl_gemm_bf16(xp, rows_total, row_offset, M, d, w13, 2 * f, h_scratch, f, nullptr, 2, stream);
    if (rc) return rc;
    return kl_gemm_bf16(h_scratch, M, 0, M, f, w2, d, y + row_offset * d, d, nullptr, 0, stream);
}
