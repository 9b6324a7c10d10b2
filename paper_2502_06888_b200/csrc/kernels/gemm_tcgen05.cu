// SPDX-License-Identifier: Apache-2.0
// K5: bf16 GEMM / grouped expert FFN on 5th-gen tensor cores (sm_100a).
//
// One CTA computes one 128 x BN output tile (optionally one K-split of it):
//   warp 0   : TMA producer  (A and B tiles, 128B swizzle, STAGES-deep ring)
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5: epilogue (tcgen05.ld TMEM -> registers -> global stores);
//              warp w owns TMEM lanes 32*(w%4) .. +31 (= tile rows).
// Pipelines: smem full/empty mbarriers between TMA and MMA, one accumulator
// barrier between MMA (tcgen05.commit) and the epilogue.
//
// Decode shapes (M = a few hundred routed rows per expert) are HBM-bound on
// the weight stream, so the host picks the tile shape / CTAs per SM / K-split
// that keeps every SM streaming weights in one wave. K-splits write fp32
// partials that a second kernel sums in fixed split order (deterministic)
// and finishes with the epilogue (bf16 store, +residual, or SwiGLU).
//
// Used for the expert FFN (compute_expert, reference schedule.cpp:355-372,
// which the reference only prices at token_count * t_c_e_per_token,
// simulator.cpp:17) and for the attention projections / LM head.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace kl {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle span
constexpr int kThreads = 192;

enum Epilogue { kStore = 0, kResidual = 1, kSwiGLU = 2, kPartial = 3 };

template <int BN, int STAGES>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = BN;  // fp32 accumulator columns (power of two >= 32)
    static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kMinBlocks = kSmemBytes * 2 <= 227 * 1024 ? 2 : 1;
};

// PAIRED: the B tile is two BN/2-row halves [W1 rows | W3 rows] of the same
// output columns (SwiGLU gate/up), read at row offsets n and b_half_rows + n.
template <int BN, int EPI, bool PAIRED, int STAGES>
__global__ void __launch_bounds__(kThreads, (Cfg<BN, STAGES>::kMinBlocks))
gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  int a_row0, int M, int kb_per_split, int b_half_rows, uint16_t* __restrict__ c, int ldc,
                  const uint16_t* __restrict__ r, float* __restrict__ ws, int ws_ld) {
    using C = Cfg<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_ready = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n_tile = blockIdx.x;
    const int m_tile = blockIdx.y;
    const int split = blockIdx.z;
    const int kb0 = split * kb_per_split;
    const int num_kb = kb_per_split;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
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
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % STAGES;
                const uint32_t phase = (i / STAGES) & 1;
                const int kc = (kb0 + i) * BK;
                mbar_wait(&empty[s], phase ^ 1);
                uint8_t* sa = smem + s * C::kStageBytes;
                uint8_t* sb = sa + C::kABytes;
                mbar_arrive_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(sa, &tmap_a, &full[s], kc, a_row);
                if constexpr (PAIRED) {
                    tma_load_2d(sb, &tmap_b, &full[s], kc, n_tile * (BN / 2));
                    tma_load_2d(sb + (BN / 2) * BK * 2, &tmap_b, &full[s], kc, b_half_rows + n_tile * (BN / 2));
                } else {
                    tma_load_2d(sb, &tmap_b, &full[s], kc, n_tile * BN);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % STAGES;
                const uint32_t phase = (i / STAGES) & 1;
                mbar_wait(&full[s], phase);
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + s * C::kStageBytes);
                const uint32_t sb = sa + C::kABytes;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // UMMA_K = 16 bf16 = 32 bytes along the swizzled row.
                    tc_mma_bf16(tmem_base, sw128_kmajor_desc(sa + k * 32), sw128_kmajor_desc(sb + k * 32), idesc,
                                (i | k) != 0);
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
        const int row = m_tile * BM + quarter * 32 + lane;
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
        const bool live = row < M;
        if constexpr (EPI == kPartial) {
            float* out = ws + (static_cast<int64_t>(split) * M + row) * ws_ld + static_cast<int64_t>(n_tile) * BN;
#pragma unroll 1
            for (int col = 0; col < BN; col += 16) {
                float v[16];
                tmem_ld16(lane_addr + col, v);
                if (live) {
                    float4* dst = reinterpret_cast<float4*>(out + col);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
        } else if constexpr (EPI == kSwiGLU) {
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

// Sum the K-split partials in split order (deterministic) and apply the
// epilogue. Each thread produces 4 consecutive output columns of one row.
template <int EPI>
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int ws_ld, int n_out, int pair_bn,
                                     uint16_t* __restrict__ c, int ldc, const uint16_t* __restrict__ r) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int quads = n_out / 4;
    if (q >= static_cast<int64_t>(M) * quads) return;
    const int m = static_cast<int>(q / quads);
    const int j = static_cast<int>(q % quads) * 4;
    const int64_t split_stride = static_cast<int64_t>(M) * ws_ld;
    float out[4];
    if constexpr (EPI == kSwiGLU) {
        const int half = pair_bn / 2;
        const int tile = j / half, w = j % half;
        const float* g = ws + static_cast<int64_t>(m) * ws_ld + static_cast<int64_t>(tile) * pair_bn + w;
        float4 ga = *reinterpret_cast<const float4*>(g);
        float4 ua = *reinterpret_cast<const float4*>(g + half);
        for (int s = 1; s < splits; ++s) {
            const float4 gb = *reinterpret_cast<const float4*>(g + s * split_stride);
            const float4 ub = *reinterpret_cast<const float4*>(g + s * split_stride + half);
            ga.x += gb.x; ga.y += gb.y; ga.z += gb.z; ga.w += gb.w;
            ua.x += ub.x; ua.y += ub.y; ua.z += ub.z; ua.w += ub.w;
        }
        const float gv[4] = {ga.x, ga.y, ga.z, ga.w}, uv[4] = {ua.x, ua.y, ua.z, ua.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = gv[i] / (1.0f + expf(-gv[i])) * uv[i];
    } else {
        const float* p = ws + static_cast<int64_t>(m) * ws_ld + j;
        float4 a = *reinterpret_cast<const float4*>(p);
        for (int s = 1; s < splits; ++s) {
            const float4 b = *reinterpret_cast<const float4*>(p + s * split_stride);
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
        if constexpr (EPI == kResidual) {
            const uint2 rv = *reinterpret_cast<const uint2*>(r + static_cast<int64_t>(m) * ldc + j);
            out[0] += bf2f(static_cast<uint16_t>(rv.x & 0xffffu));
            out[1] += bf2f(static_cast<uint16_t>(rv.x >> 16));
            out[2] += bf2f(static_cast<uint16_t>(rv.y & 0xffffu));
            out[3] += bf2f(static_cast<uint16_t>(rv.y >> 16));
        }
    }
    *reinterpret_cast<uint2*>(c + static_cast<int64_t>(m) * ldc + j) = make_uint2(pack2(out[0], out[1]), pack2(out[2], out[3]));
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
    const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return res == CUDA_SUCCESS ? 0 : KL_EINVAL;
}

struct Launch {
    const uint16_t* a;
    int64_t a_rows, row_offset;
    int M, K;
    const uint16_t* b;
    int64_t b_rows;
    int n_tiles, b_half_rows;
    uint16_t* c;
    int ldc;
    const uint16_t* r;
    int splits;
    float* ws;
    int ws_ld;
};

template <int BN, int EPI, bool PAIRED, int STAGES>
int launch(const Launch& L, cudaStream_t stream) {
    using C = Cfg<BN, STAGES>;
    CUtensorMap ma, mb;
    int rc = make_map(&ma, L.a, L.a_rows, L.K, BM);
    if (rc) return rc;
    rc = make_map(&mb, L.b, L.b_rows, L.K, PAIRED ? BN / 2 : BN);
    if (rc) return rc;
    static bool configured = false;  // per template instance
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI, PAIRED, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
        configured = true;
    }
    const dim3 grid(L.n_tiles, (L.M + BM - 1) / BM, L.splits);
    gemm_bf16_tcgen05<BN, EPI, PAIRED, STAGES><<<grid, kThreads, C::kSmemBytes, stream>>>(
        ma, mb, static_cast<int>(L.row_offset), L.M, L.K / BK / L.splits, L.b_half_rows, L.c, L.ldc, L.r, L.ws,
        L.ws_ld);
    return check_launch();
}

template <int EPI>
int reduce(const Launch& L, int n_out, int pair_bn, cudaStream_t stream) {
    const int64_t threads = static_cast<int64_t>(L.M) * (n_out / 4);
    splitk_reduce_kernel<EPI><<<static_cast<int>((threads + 255) / 256), 256, 0, stream>>>(
        L.ws, L.splits, L.M, L.ws_ld, n_out, pair_bn, L.c, L.ldc, L.r);
    return check_launch();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kSMs = 148;

// Split count for a weight-streaming (small-M) GEMM: enough CTAs for two per
// SM in one wave, at least 16 k-blocks (1024 of K) per split, K-blocks
// divisible by the split count, and within the caller's workspace.
int choose_splits(int tiles, int kb, int M, int ws_cols, int64_t ws_bytes) {
    int best = 1;
    for (int s = 1; s <= 16; ++s) {
        if (kb % s != 0 || kb / s < 16) continue;
        if (static_cast<int64_t>(s) * M * ws_cols * 4 > ws_bytes) break;
        if (tiles * s <= 2 * kSMs) best = s;
    }
    return best;
}

}  // namespace
}  // namespace kl

extern "C" int64_t kl_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
    using namespace kl;
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    const int m_tiles = (M + BM - 1) / BM;
    const int tiles = (N / 128) * m_tiles;
    const int s = choose_splits(tiles, K / BK, M, N, INT64_MAX);
    (void)epilogue;
    return s > 1 ? static_cast<int64_t>(s) * M * N * 4 : 0;
}

extern "C" int kl_gemm_bf16(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b,
                            int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace,
                            int64_t workspace_bytes, cudaStream_t stream) {
    using namespace kl;
    if (M < 0 || K <= 0 || N <= 0 || a == nullptr || b == nullptr || c == nullptr) return KL_EINVAL;
    if (M == 0) return KL_OK;
    if (K % BK != 0 || N % 64 != 0 || !aligned16(a) || !aligned16(b) || !aligned16(c) || ldc % 8 != 0)
        return KL_EINVAL;
    if (row_offset < 0 || row_offset + M > a_rows || row_offset > INT32_MAX) return KL_EINVAL;
    if (epilogue < 0 || epilogue > 2) return KL_EINVAL;
    if (epilogue == kResidual && (r == nullptr || !aligned16(r))) return KL_EINVAL;
    if (epilogue == kSwiGLU && N % 256 != 0) return KL_EINVAL;
    if (workspace != nullptr && !aligned16(workspace)) return KL_EINVAL;
    const int m_tiles = (M + BM - 1) / BM;
    const int kb = K / BK;
    Launch L{a, a_rows, row_offset, M, K, b, N, 0, 0, c, ldc, r, 1, static_cast<float*>(workspace), N};
    const bool small_m = m_tiles <= 2 && N % 128 == 0;  // weight-streaming regime (decode)
    if (small_m) {
        // 128-wide tiles (activation:weight smem traffic 1:1), 2 CTAs per SM,
        // K-split until the grid fills both CTA slots of every SM.
        L.n_tiles = N / 128;
        L.splits = workspace ? choose_splits(L.n_tiles * m_tiles, kb, M, N, workspace_bytes) : 1;
        const bool paired = epilogue == kSwiGLU;
        L.b_half_rows = paired ? N / 2 : 0;
        if (L.splits > 1) {
            int rc = paired ? launch<128, kPartial, true, 3>(L, stream) : launch<128, kPartial, false, 3>(L, stream);
            if (rc) return rc;
            if (epilogue == kSwiGLU) return reduce<kSwiGLU>(L, N / 2, 128, stream);
            if (epilogue == kResidual) return reduce<kResidual>(L, N, 128, stream);
            return reduce<kStore>(L, N, 128, stream);
        }
        if (epilogue == kSwiGLU) return launch<128, kSwiGLU, true, 3>(L, stream);
        if (epilogue == kResidual) return launch<128, kResidual, false, 3>(L, stream);
        return launch<128, kStore, false, 3>(L, stream);
    }
    // Compute-bound regime (prefill / large M): 256-wide tiles, deep pipeline.
    if (epilogue == kSwiGLU) {
        L.n_tiles = N / 256;
        L.b_half_rows = N / 2;
        return launch<256, kSwiGLU, true, 4>(L, stream);
    }
    if (N % 256 == 0) {
        L.n_tiles = N / 256;
        return epilogue == kResidual ? launch<256, kResidual, false, 4>(L, stream)
                                     : launch<256, kStore, false, 4>(L, stream);
    }
    L.n_tiles = N / 64;
    return epilogue == kResidual ? launch<64, kResidual, false, 6>(L, stream) : launch<64, kStore, false, 6>(L, stream);
}

extern "C" int kl_expert_ffn(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d, int f,
                             const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch, uint16_t* y,
                             void* workspace, int64_t workspace_bytes, cudaStream_t stream) {
    if (M == 0) return KL_OK;
    if (y == nullptr || h_scratch == nullptr) return KL_EINVAL;
    int rc = kl_gemm_bf16(xp, rows_total, row_offset, M, d, w13, 2 * f, h_scratch, f, nullptr, 2, workspace,
                          workspace_bytes, stream);
    if (rc) return rc;
    return kl_gemm_bf16(h_scratch, M, 0, M, f, w2, d, y + row_offset * d, d, nullptr, 0, workspace, workspace_bytes,
                        stream);
}
