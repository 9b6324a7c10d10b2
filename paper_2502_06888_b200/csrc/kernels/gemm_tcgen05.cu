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
#include <atomic>
#include <mutex>

#include "common.cuh"
#include "tma_host.cuh"

namespace kl {
extern int g_pdl;  // kl_tune(KL_TUNE_PDL, ...): programmatic dependent launch (abi.cu)
// kl_stamp_next_launch: the next GEMM this host thread launches marks the op
// start itself (one kernel fewer in the op's launch chain).
thread_local unsigned long long* t_next_start = nullptr;
namespace {
// kl_tune(KL_TUNE_STREAM_HINT, ...): L2 policy hints on weight loads: 1 = weights
// evict-first / activations evict-last, 2 = weights evict-last, 0 = none.
int g_stream_hint = 1;

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
                  const uint16_t* __restrict__ r, float* __restrict__ ws, int ws_ld, int b_hint) {
    pdl_enter();
    using C = Cfg<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_ready = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // Grouped raster: CTAs launched together cover a block of kGroupM
    // m-tiles x a few n-tiles (m fastest), so both the activation and the
    // weight tiles of a wave are reused from L2 instead of re-streaming the
    // whole weight matrix once per row of m-tiles.
    int n_tile = blockIdx.x, m_tile = blockIdx.y;
    if (gridDim.y > 1) {
        constexpr int kGroupM = 16;
        const int lin = blockIdx.y * gridDim.x + blockIdx.x;
        const int per_group = kGroupM * gridDim.x;
        const int first_m = lin / per_group * kGroupM;
        const int group_m = min(kGroupM, static_cast<int>(gridDim.y) - first_m);
        const int within = lin % per_group;
        m_tile = first_m + within % group_m;
        n_tile = within / group_m;
    }
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
            // Weights: no hint (1), L2 evict-last (2) when the caller reuses them soon.
            const uint64_t pol_b = l2_policy_evict_last();
            const bool hb = b_hint == 2;
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % STAGES;
                const uint32_t phase = (i / STAGES) & 1;
                const int kc = (kb0 + i) * BK;
                mbar_wait(&empty[s], phase ^ 1);
                uint8_t* sa = smem + s * C::kStageBytes;
                uint8_t* sb = sa + C::kABytes;
                mbar_arrive_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(sa, &tmap_a, &full[s], kc, a_row);
                // Weights through a 3D (64, rows, k-blocks) view: the same
                // smem image for row-major and K-blocked weight layouts.
                if constexpr (PAIRED) {
                    tma_load_3d_k(sb, &tmap_b, &full[s], n_tile * (BN / 2), kc / BK, pol_b, hb);
                    tma_load_3d_k(sb + (BN / 2) * BK * 2, &tmap_b, &full[s], b_half_rows + n_tile * (BN / 2), kc / BK,
                                  pol_b, hb);
                } else {
                    tma_load_3d_k(sb, &tmap_b, &full[s], n_tile * BN, kc / BK, pol_b, hb);
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

// Persistent form of the compute-bound (prefill) GEMM: one CTA per SM walks
// its tiles (stride gridDim.x over the grouped raster order), the TMA ring
// runs continuously across tiles, and two TMEM accumulators alternate so a
// tile's epilogue (SwiGLU / residual / store) overlaps the next tile's MMAs.
template <int BN, int EPI, bool PAIRED, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
gemm_persistent_tcgen05(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        int a_row0, int M, int num_kb, int b_half_rows, int n_tiles, int m_tiles,
                        uint16_t* __restrict__ c, int ldc, const uint16_t* __restrict__ r) {
    using C = Cfg<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    constexpr uint32_t kCols = 2 * BN;    // two accumulators

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int total = n_tiles * m_tiles;
    auto tile_of = [&](int lin, int& n_tile, int& m_tile) {
        constexpr int kGroupM = 16;
        const int per_group = kGroupM * n_tiles;
        const int first_m = lin / per_group * kGroupM;
        const int group_m = min(kGroupM, m_tiles - first_m);
        const int within = lin % per_group;
        m_tile = first_m + within % group_m;
        n_tile = within / group_m;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, kCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int lin = blockIdx.x; lin < total; lin += gridDim.x) {
                int n_tile, m_tile;
                tile_of(lin, n_tile, m_tile);
                const int a_row = a_row0 + m_tile * BM;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* sa = smem + s * C::kStageBytes;
                    uint8_t* sb = sa + C::kABytes;
                    mbar_arrive_expect_tx(&full[s], C::kStageBytes);
                    tma_load_2d(sa, &tmap_a, &full[s], kb * BK, a_row);
                    if constexpr (PAIRED) {
                        tma_load_3d_k(sb, &tmap_b, &full[s], n_tile * (BN / 2), kb, 0, false);
                        tma_load_3d_k(sb + (BN / 2) * BK * 2, &tmap_b, &full[s], b_half_rows + n_tile * (BN / 2), kb, 0,
                                      false);
                    } else {
                        tma_load_3d_k(sb, &tmap_b, &full[s], n_tile * BN, kb, 0, false);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
            int it = 0, lt = 0;
            for (int lin = blockIdx.x; lin < total; lin += gridDim.x, ++lt) {
                const int b = lt & 1;
                mbar_wait(&acc_empty[b], ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t acc = tmem_base + b * BN;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * C::kStageBytes);
                    const uint32_t sb = sa + C::kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc_mma_bf16(acc, sw128_kmajor_desc(sa + k * 32), sw128_kmajor_desc(sb + k * 32), idesc,
                                    (kb | k) != 0);
                    tc_commit(&empty[s]);
                }
                tc_commit(&acc_full[b]);
            }
        }
        __syncwarp();
    } else {
        const int quarter = warp & 3;
        int lt = 0;
        for (int lin = blockIdx.x; lin < total; lin += gridDim.x, ++lt) {
            int n_tile, m_tile;
            tile_of(lin, n_tile, m_tile);
            const int b = lt & 1;
            mbar_wait(&acc_full[b], (lt >> 1) & 1);
            tc_fence_after();
            const int row = m_tile * BM + quarter * 32 + lane;
            const uint32_t lane_addr = tmem_base + b * BN + (static_cast<uint32_t>(quarter * 32) << 16);
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
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kCols);
    }
}

// Sum the K-split partials in split order (deterministic) and apply the
// epilogue. Each thread produces 4 consecutive output columns of one row.
template <int EPI>
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int ws_ld, int n_out, int pair_bn,
                                     uint16_t* __restrict__ c, int ldc, const uint16_t* __restrict__ r) {
    pdl_enter();
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

// ------------------------------------------- weight-streaming (decode) GEMM --
// Decode-shaped GEMMs (M <= 256 activation rows against a weight matrix of
// tens to hundreds of MB) are bound by reading the weights once from HBM.
// Layout choice ("swap AB"): the MMA's M side is the weights (128 output
// features per UMMA, read by TMA once), its N side the activation rows
// padded to NP (multiple of 16), so one accumulator covers every row and no
// weight byte is read twice however many rows the expert got. NMMA weight
// sub-tiles (1 or 2) share each activation tile, halving activation L2
// traffic when 2; for SwiGLU the pair is (W1 rows, W3 rows) of the same 128
// features, so gate and up land in the same TMEM lane and the epilogue needs
// no exchange.
//
// Work split ("stream-K"): the (tile, k-block) space is cut into gridDim
// contiguous, equal ranges, one persistent CTA per SM, so every SM streams
// the same number of weight bytes (no partial last wave). A tile cut by a
// range boundary is finished by its "owner" — the CTA holding the tile's
// last k-block — which adds the fp32 partials of the lower-numbered CTAs
// that hold its earlier k-blocks, in ascending CTA order (deterministic).
// Each CTA walks its tiles last-to-first, so the partial it contributes is
// published first and the tile it owns is finished last: owners rarely wait,
// and they only ever wait on lower-numbered (earlier-dispatched) CTAs, which
// guarantees forward progress.
constexpr int kStreamThreads = 192;
constexpr int kWRows = 128;  // weight rows per UMMA (M)
constexpr int kWTileBytes = kWRows * BK * 2;

struct StreamArgs {
    int M;          // valid activation rows
    int NP;         // MMA N: rows padded to a multiple of 16 (<= 256)
    int acc_stride; // TMEM columns between the NMMA accumulators
    int nbuf;       // TMEM accumulator sets (2 = epilogue overlaps the next segment's MMAs)
    int KB;         // k-blocks per tile
    int units;      // n_tiles * KB
    int half_rows;  // SwiGLU: first W3 row inside B
    int stages;
    uint16_t* c;
    int ldc;
    const uint16_t* r;
    float* ws;        // [grid] partial slots, each [NMMA][NP/16][4][128] float4
    uint32_t* flags;  // [grid] publish epochs
    uint32_t epoch;
    uint32_t tmem_cols;
    int hint;   // 1 = L2 cache-policy hints on the TMA loads
    int pdl;    // launched with programmatic stream serialization
    int ks;     // k-blocks per stage: 2 = one 3D TMA box covers two 64-column k-blocks (larger copies)
    int debug;  // benchmarking only: bit0 skip MMAs, bit1 skip epilogue work
    int split;        // > 0: tile-aligned splits, S per tile (G = tiles x S); 0: stream-K ranges
    unsigned long long* t_start;  // op start mark: %globaltimer once the previous grid is done (kl_stamp_next_launch)
    unsigned long long* t_end;    // op end mark: written by the last CTA to finish (kl_stamp_end_next_launch)
    unsigned* end_cnt;
    // Deferred split reduction (kStore, NMMA 1, tile-aligned splits): every CTA
    // writes its fp32 accumulator to defer[split][row][feature] (row pitch
    // defer_ld) and the consumer sums the splits; no flags, no fixup.
    float* defer;
    int64_t defer_split_elems;
    int defer_ld;
    // Fused RoPE + KV append (QKV projection, one 128-row weight tile = one
    // head of hd 128): rows [q heads | k heads | v heads], NeoX pairs.
    const float2* rope_tab;  // [M][64] (cos, sin) per row and frequency; nullptr = plain store
    const int32_t* rope_pos;
    const int32_t* rope_seq;
    uint16_t* kc;
    uint16_t* vc;
    int Hq, Hkv, cap, sink, chunk_last_pos;
    int stage_off;    // > 0: byte offset of a dedicated output staging region (owner adds the
                      // landed partials while it reads TMEM for the epilogue; no TMEM store-back)
    const uint8_t* q4;  // Q4 variant: weights in the tiled 4-bit layout (kQ4Chunk bytes per 128x64 tile)
};

// 4-bit weights ("Q4T", the reference's HQQ format, quant.cpp:197-252, with
// its groups of 64 laid out per 128-row x 64-column tile): per tile 128 rows
// x 32 bytes of little-endian nibble codes, then 128 fp16 scales, then 128
// fp16 zeros; w = scale * (code - zero). Tiles ordered (row tile, k-block).
constexpr int kQ4Chunk = kWRows * 32 + kWRows * 2 * 2;  // 4608 bytes per 8192 weights

__device__ unsigned long long g_stream_trace[256][12];  // debug & 128: per-CTA phase timestamps (ns)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define STREAM_TRACE(slot) \
    do { if (p.debug & 128) g_stream_trace[blockIdx.x][slot] = gtimer(); } while (0)

__device__ __forceinline__ int range_begin(int c, int units, int G) {
    return static_cast<int>(static_cast<int64_t>(c) * units / G);
}
// First unit of CTA c. With tile-aligned splits (p.split = S > 0, G = tiles
// x S) each tile's k-blocks are cut into S ranges, the last (the owner's)
// taking the remainder when S does not divide KB.
__device__ __forceinline__ int unit_begin(const StreamArgs& p, int c, int G) {
    if (p.split <= 0) return range_begin(c, p.units, G);
    const int t = c / p.split, j = c % p.split;
    return t * p.KB + j * (p.KB / p.split);
}


// 1D bulk copy global -> shared (async proxy), completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <int EPI>
__device__ __forceinline__ float epi_value(const float (&acc)[2][16], int j, int i) {
    if constexpr (EPI == kSwiGLU) {
        const float g = acc[0][i], u = acc[1][i];
        return __fdividef(g, 1.0f + __expf(-g)) * u;
    } else {
        return acc[j][i];
    }
}

// One 16-byte vector (8 features) of a staged QKV row: rotate q / k heads
// with the row's (cos, sin) table (same rope_lo / rope_hi as the RoPE
// kernels), store to the QKV output, and append k / v heads to the cache.
__device__ __forceinline__ void rope_row_store(const StreamArgs& p, const uint16_t* stage, int row, int x, int head,
                                               uint16_t* o) {
    const uint4 v = *reinterpret_cast<const uint4*>(stage + row * kWRows + x * 8);
    uint4 r = v;
    const int rot = p.Hq + p.Hkv;
    if (head < rot) {
        const uint4 w = *reinterpret_cast<const uint4*>(stage + row * kWRows + (x ^ 8) * 8);
        const float2* tb = p.rope_tab + static_cast<int64_t>(row) * (kWRows / 2) + (x & 7) * 8;
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w}, ww[4] = {w.x, w.y, w.z, w.w};
        uint32_t rr[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float out2[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float2 t = __ldg(tb + 2 * e + h);
                const float self = bf2f(static_cast<uint16_t>(h ? vv[e] >> 16 : vv[e] & 0xffffu));
                const float other = bf2f(static_cast<uint16_t>(h ? ww[e] >> 16 : ww[e] & 0xffffu));
                out2[h] = x < 8 ? rope_lo(self, other, t.x, t.y) : rope_hi(other, self, t.x, t.y);
            }
            rr[e] = pack2(out2[0], out2[1]);
        }
        r = make_uint4(rr[0], rr[1], rr[2], rr[3]);
    }
    *reinterpret_cast<uint4*>(o) = r;
    if (head >= p.Hq) {
        const int pp = p.rope_pos[row];
        if (p.chunk_last_pos < 0 || pp < p.sink || pp > p.chunk_last_pos - (p.cap - p.sink)) {
            const int64_t crow = (static_cast<int64_t>(p.rope_seq[row]) * p.cap + kv_slot_of(pp, p.cap, p.sink)) *
                                 p.Hkv * kWRows;
            uint16_t* dst = head < rot ? p.kc + crow + static_cast<int64_t>(head - p.Hq) * kWRows
                                       : p.vc + crow + static_cast<int64_t>(head - rot) * kWRows;
            *reinterpret_cast<uint4*>(dst + x * 8) = r;
        }
    }
}

template <int EPI, int NMMA, bool Q4>
__global__ void __launch_bounds__(kStreamThreads, 1)
gemm_stream_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, int a_row0,
                   const StreamArgs p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = p.ks * (NMMA * kWTileBytes + p.NP * BK * 2);
    const int wbytes = p.ks * kWTileBytes;  // one weight sub-tile's k-chunks in a stage
    const int ring_bytes = p.stages * stage_bytes;
    constexpr int kRawStage = NMMA * kQ4Chunk;
    uint8_t* raw = smem + ring_bytes;  // Q4: packed tiles land here, dequantised into the ring
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + (Q4 ? p.stages * kRawStage : 0));
    uint64_t* empty = full + p.stages;
    uint64_t* acc_full = empty + p.stages;  // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2]
    uint64_t* part_bar = acc_empty + 2;
    uint64_t* raw_full = part_bar + 1;  // [stages] (Q4)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_full + p.stages);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, cta = blockIdx.x;
    const int KB = p.KB;
    const int u0 = unit_begin(p, cta, G), u1 = unit_begin(p, cta + 1, G);
    const int t_hi = u1 > u0 ? (u1 - 1) / KB : 0, t_lo = u1 > u0 ? u0 / KB : 1;  // tiles walked t_hi .. t_lo
    const int buf_cols = NMMA * p.acc_stride;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], Q4 ? 5 : 1);  // Q4: + one arrival per dequantising warp
            mbar_init(&empty[s], 1);
            if (Q4) mbar_init(&raw_full[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_init(part_bar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x == 0) STREAM_TRACE(0);
    if (p.pdl) griddep_launch_dependents();
    if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = p.hint == 2 ? l2_policy_evict_last() : l2_policy_evict_first();
            const uint64_t pol_x = l2_policy_evict_last();
            const bool hint = p.hint != 0;
            // Programmatic dependent launch: the weights do not depend on the
            // previous kernel, so the first `stages` weight tiles are issued
            // before griddepcontrol.wait; activations, outputs and the
            // workspace are touched only after it.
            bool waited = !p.pdl;
            int it = 0, pending_x = 0;
            auto load_x = [&](int s_, int kb_) {
                uint8_t* sx = smem + s_ * stage_bytes + NMMA * wbytes;
                if (p.ks > 1)
                    tma_load_3d_k(sx, &tmap_x, &full[s_], a_row0, kb_ * p.ks, pol_x, hint);
                else if (hint)
                    tma_load_2d_hint(sx, &tmap_x, &full[s_], kb_ * BK, a_row0, pol_x);
                else
                    tma_load_2d(sx, &tmap_x, &full[s_], kb_ * BK, a_row0);
            };
            int xkb[16];  // k-block of each stage issued before the wait
            for (int t = t_hi; t >= t_lo; --t) {
                const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % p.stages;
                    if (!waited && it >= p.stages) {
                        griddep_wait();
                        waited = true;
                        for (int i = 0; i < pending_x; ++i) load_x(i, xkb[i]);
                    }
                    mbar_wait(&empty[s], ((it / p.stages) & 1) ^ 1);
                    uint8_t* sw = smem + s * stage_bytes;
                    mbar_arrive_expect_tx(&full[s], Q4 ? p.NP * BK * 2 : stage_bytes);
                    if constexpr (Q4) mbar_arrive_expect_tx(&raw_full[s], kRawStage);
#pragma unroll
                    for (int j = 0; j < NMMA; ++j) {
                        const int row = EPI == kSwiGLU ? (j == 0 ? t * kWRows : p.half_rows + t * kWRows)
                                                       : (t * NMMA + j) * kWRows;
                        if constexpr (Q4) {
                            const uint8_t* src = p.q4 + (static_cast<int64_t>(row / kWRows) * KB + kb) * kQ4Chunk;
                            bulk_g2s(raw + s * kRawStage + j * kQ4Chunk, src, kQ4Chunk, &raw_full[s]);
                        } else {
                            // 3D (64, rows, k-blocks) view of the weights, p.ks
                            // k-blocks per box: row-major or K-blocked layout.
                            tma_load_3d_k(sw + j * wbytes, &tmap_w, &full[s], row, kb * p.ks, pol_w, hint);
                        }
                    }
                    if (waited) {
                        load_x(s, kb);
                    } else {
                        xkb[pending_x++] = kb;
                    }
                }
            }
            if (!waited) {
                griddep_wait();
                for (int i = 0; i < pending_x; ++i) load_x(i, xkb[i]);
            }
        }
        if (p.pdl) griddep_wait();  // every thread: outputs/workspace only after the previous grid
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16_f32(kWRows, p.NP);
            int it = 0, seg = 0;
            for (int t = t_hi; t >= t_lo; --t, ++seg) {
                const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
                const int b = p.nbuf == 2 ? (seg & 1) : 0, use = p.nbuf == 2 ? (seg >> 1) : seg;
                mbar_wait(&acc_empty[b], (use & 1) ^ 1);  // epilogue drained this accumulator set
                tc_fence_after();
                const uint32_t acc0 = tmem_base + b * buf_cols;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % p.stages;
                    mbar_wait(&full[s], (it / p.stages) & 1);
                    if (it == 0) STREAM_TRACE(1);
                    tc_fence_after();
                    const uint32_t sw = smem_u32(smem + s * stage_bytes);
                    const uint32_t sx = sw + NMMA * wbytes;
                    if (!(p.debug & 1))
                        for (int kk = 0; kk < p.ks; ++kk)
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
                                for (int j = 0; j < NMMA; ++j)
                                    tc_mma_bf16(acc0 + j * p.acc_stride,
                                                sw128_kmajor_desc(sw + j * wbytes + kk * kWTileBytes + k * 32),
                                                sw128_kmajor_desc(sx + kk * p.NP * BK * 2 + k * 32), idesc,
                                                (kb > kb0 || kk > 0 || k > 0) ? 1u : 0u);
                    tc_commit(&empty[s]);
                }
                tc_commit(&acc_full[b]);
            }
            STREAM_TRACE(2);
        }
        __syncwarp();
    } else {
        if (p.pdl) griddep_wait();
        if (p.t_start != nullptr && blockIdx.x == 0 && threadIdx.x == 64) *p.t_start = gtimer();
        const int quarter = warp & 3;
        const int frow = quarter * 32 + lane;  // feature row inside a 128-row sub-tile
        const int etid = threadIdx.x - 64;     // 0..127 across the epilogue warps
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const int cols = (p.M + 15) & ~15;  // token columns worth reading
        const int nch = p.NP / 16;
        const int slot_f4 = NMMA * kWRows * (p.NP / 4);  // float4 per partial slot
        auto slot4 = [&](int q) { return reinterpret_cast<float4*>(p.ws) + static_cast<int64_t>(q) * slot_f4; };
        int seg = 0, dq_it = 0;
        for (int t = t_hi; t >= t_lo; --t, ++seg) {
            const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
            const int b = p.nbuf == 2 ? (seg & 1) : 0, use = p.nbuf == 2 ? (seg >> 1) : seg;
            if constexpr (Q4) {
                // Dequantise this segment's stages into the bf16 ring (thread = weight row),
                // written in the 128B-swizzled K-major layout the MMA descriptors expect.
                for (int kb = kb0; kb < kb1; ++kb, ++dq_it) {
                    const int s = dq_it % p.stages;
                    mbar_wait(&raw_full[s], (dq_it / p.stages) & 1);
#pragma unroll
                    for (int j = 0; j < NMMA; ++j) {
                        const uint8_t* rc = raw + s * kRawStage + j * kQ4Chunk;
                        const uint4 c0 = *reinterpret_cast<const uint4*>(rc + frow * 32);
                        const uint4 c1 = *reinterpret_cast<const uint4*>(rc + frow * 32 + 16);
                        const float sc = __half2float(__ushort_as_half(*reinterpret_cast<const uint16_t*>(rc + kWRows * 32 + frow * 2)));
                        const float zr = __half2float(
                            __ushort_as_half(*reinterpret_cast<const uint16_t*>(rc + kWRows * 32 + kWRows * 2 + frow * 2)));
                        const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
                        uint8_t* wrow = smem + s * stage_bytes + j * kWTileBytes + frow * 128;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            uint32_t pk[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __fmul_rn(sc, __fsub_rn(static_cast<float>((cw[u] >> (8 * e)) & 15u), zr));
                                const float hi = __fmul_rn(sc, __fsub_rn(static_cast<float>((cw[u] >> (8 * e + 4)) & 15u), zr));
                                pk[e] = pack2(lo, hi);
                            }
                            *reinterpret_cast<uint4*>(wrow + ((u ^ (frow & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[s]);
                }
            }
            mbar_wait(&acc_full[b], use & 1);
            tc_fence_after();
            const uint32_t acc0 = tmem_base + lane_off + b * buf_cols;
            const bool has_last = kb1 == KB;
            if (p.debug & 2) {
            } else if (p.defer != nullptr) {
                float* dst = p.defer + static_cast<int64_t>(cta % p.split) * p.defer_split_elems +
                             static_cast<int64_t>(t) * kWRows + frow;
                for (int col = 0; col < cols; col += 16) {
                    float v[16];
                    tmem_ld16(acc0 + col, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (col + i < p.M) __stcg(dst + static_cast<int64_t>(col + i) * p.defer_ld, v[i]);
                }
            } else if (!has_last) {
                // Contributor: publish the fp32 partial of this tile. Slot
                // layout [j][16-column chunk][float4 i][feature row] so each
                // warp store / load is 512 contiguous bytes.
                if (etid == 0) STREAM_TRACE(8);
                float4* slot = slot4(cta);
                for (int j = 0; j < NMMA; ++j) {
                    for (int col = 0; col < cols; col += 32) {
                        // 32 columns per TMEM load (one wait), the second 16 only if live.
                        float v[32];
                        tmem_ld32(acc0 + j * p.acc_stride + col, v);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (col + 16 * h >= cols) break;
                            float4* dst = slot + (static_cast<int64_t>(j * nch + (col >> 4) + h) * 4) * kWRows + frow;
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                __stcg(dst + i * kWRows, make_float4(v[16 * h + 4 * i], v[16 * h + 4 * i + 1],
                                                                     v[16 * h + 4 * i + 2], v[16 * h + 4 * i + 3]));
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);
                __threadfence();
                named_bar_sync(1, 128);
                if (etid == 0) st_release_gpu(p.flags + cta, p.epoch);
                if (etid == 0) STREAM_TRACE(9);
                continue;
            } else if (t != t_lo) {
                // A whole tile in the middle of the range (only when a range
                // spans more than a tile): direct, uncoalesced stores. (The
                // host never lets the fused RoPE epilogue reach this path.)
                if (p.rope_tab != nullptr) __trap();
                for (int col = 0; col < cols; col += 16) {
                    float acc[2][16];
#pragma unroll
                    for (int j = 0; j < NMMA; ++j) tmem_ld16(acc0 + j * p.acc_stride + col, acc[j]);
#pragma unroll
                    for (int j = 0; j < (EPI == kSwiGLU ? 1 : NMMA); ++j) {
                        const int64_t feat = static_cast<int64_t>(EPI == kSwiGLU ? t : t * NMMA + j) * kWRows + frow;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            if (col + i >= p.M) continue;
                            float v = epi_value<EPI>(acc, j, i);
                            uint16_t* o = p.c + static_cast<int64_t>(col + i) * p.ldc + feat;
                            if constexpr (EPI == kResidual) v += bf2f(p.r[static_cast<int64_t>(col + i) * p.ldc + feat]);
                            *o = f2bf(v);
                        }
                    }
                }
            } else {
                // Last tile walked (ring idle from here on): owner fixup,
                // then the epilogue staged through shared memory.
                if (etid == 0) STREAM_TRACE(3);
                int fused_nq = 0;  // contributors' partials landed in the ring, added in the epilogue pass
                if (kb0 > 0) {
                    int c_lo = cta - 1;
                    while (c_lo > 0 && unit_begin(p, c_lo, G) > t * KB) --c_lo;
                    if (p.stage_off > 0 && (cta - c_lo) * slot_f4 * 16 <= ring_bytes) {
                        // Every partial lands at once; the epilogue below adds
                        // them to the accumulator it reads (own partial first,
                        // then ascending CTA, as the TMEM fixup would).
                        const int slot_bytes = slot_f4 * 16;
                        fused_nq = cta - c_lo;
                        if (etid < 32) {
                            // One lane per contributor: each polls its own flag and
                            // pulls that partial as soon as it is published.
                            if (etid == 0) mbar_arrive_expect_tx(part_bar, static_cast<uint32_t>(fused_nq * slot_bytes));
                            __syncwarp();
                            for (int qi = etid; qi < fused_nq; qi += 32) {
                                while (ld_relaxed_gpu(p.flags + c_lo + qi) != p.epoch) {
                                }
                                fence_acq_rel_gpu();
                                asm volatile("fence.proxy.async.global;" ::: "memory");
                                for (int off = 0; off < slot_bytes; off += 32768)
                                    bulk_g2s(smem + qi * slot_bytes + off,
                                             reinterpret_cast<const uint8_t*>(slot4(c_lo + qi)) + off,
                                             static_cast<uint32_t>(min(32768, slot_bytes - off)), part_bar);
                            }
                        }
                        if (etid == 0) STREAM_TRACE(4);
                        mbar_wait(part_bar, 0);
                        if (etid == 0) STREAM_TRACE(5);
                    } else if (slot_f4 * 16 <= ring_bytes) {
                    const int slot_bytes = slot_f4 * 16;
                    const int per_batch = max(1, ring_bytes / slot_bytes);
                    int phase = 0;
                    for (int q0 = c_lo; q0 < cta; q0 += per_batch, phase ^= 1) {
                        const int nq = min(per_batch, cta - q0);
                        if (etid == 0) {
                            for (int q = q0; q < q0 + nq; ++q)
                                while (ld_relaxed_gpu(p.flags + q) != p.epoch) {
                                }
                            fence_acq_rel_gpu();
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            mbar_arrive_expect_tx(part_bar, static_cast<uint32_t>(nq * slot_bytes));
                            for (int q = 0; q < nq; ++q)
                                for (int off = 0; off < slot_bytes; off += 32768)
                                    bulk_g2s(smem + q * slot_bytes + off,
                                             reinterpret_cast<const uint8_t*>(slot4(q0 + q)) + off,
                                             static_cast<uint32_t>(min(32768, slot_bytes - off)), part_bar);
                        }
                        if (etid == 0) STREAM_TRACE(4);
                        mbar_wait(part_bar, phase);
                        if (etid == 0) STREAM_TRACE(5);
                        const float4* land = reinterpret_cast<const float4*>(smem);
                        for (int j = 0; j < NMMA; ++j)
                            for (int col = 0; col < cols; col += 16) {
                                float v[16];
                                tmem_ld16(acc0 + j * p.acc_stride + col, v);
                                for (int q = 0; q < nq; ++q) {
                                    const float4* src =
                                        land + static_cast<int64_t>(q) * slot_f4 +
                                        (static_cast<int64_t>(j * nch + (col >> 4)) * 4) * kWRows + frow;
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        const float4 w = src[i * kWRows];
                                        v[4 * i] += w.x;
                                        v[4 * i + 1] += w.y;
                                        v[4 * i + 2] += w.z;
                                        v[4 * i + 3] += w.w;
                                    }
                                }
                                tmem_st16(acc0 + j * p.acc_stride + col, v);
                            }
                        named_bar_sync(1, 128);  // landing buffer free before the next batch
                    }
                                    } else {
                    // Contributors' partials land in the idle ring in 8 KB units
                    // (one accumulator x 16 columns each), as many per batch as fit,
                    // ordered (accumulator, column chunk, contributor): each
                    // element adds its partials in ascending CTA order with one
                    // TMEM load/store per run of units on the same columns.
                    constexpr int kUnitF4 = 4 * kWRows;
                    constexpr int kUnitBytes = kUnitF4 * 16;
                    const int nu = cols / 16, nq = cta - c_lo;
                    const int total = NMMA * nu * nq;
                    const int per_batch = max(1, ring_bytes / kUnitBytes);
                    if (etid == 0) {
                        for (int q = c_lo; q < cta; ++q)
                            while (ld_relaxed_gpu(p.flags + q) != p.epoch) {
                            }
                        fence_acq_rel_gpu();
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    int phase = 0;
                    for (int w0 = 0; w0 < total; w0 += per_batch, phase ^= 1) {
                        const int nw = min(per_batch, total - w0);
                        if (etid == 0) {
                            mbar_arrive_expect_tx(part_bar, static_cast<uint32_t>(nw * kUnitBytes));
                            for (int w = w0; w < w0 + nw; ++w) {
                                const int jc = w / nq, q = c_lo + w % nq;
                                bulk_g2s(smem + (w - w0) * kUnitBytes, slot4(q) + static_cast<int64_t>((jc / nu) * nch + jc % nu) * kUnitF4,
                                         kUnitBytes, part_bar);
                            }
                        }
                        if (etid == 0) STREAM_TRACE(4);
                        mbar_wait(part_bar, phase);
                        if (etid == 0) STREAM_TRACE(5);
                        const float4* land = reinterpret_cast<const float4*>(smem);
                        float v[16];
                        int cur = -1;
                        for (int w = w0; w < w0 + nw; ++w) {
                            const int jc = w / nq;
                            const uint32_t taddr = acc0 + (jc / nu) * p.acc_stride + (jc % nu) * 16;
                            if (jc != cur) {
                                if (cur >= 0) tmem_st16(acc0 + (cur / nu) * p.acc_stride + (cur % nu) * 16, v);
                                tmem_ld16(taddr, v);
                                cur = jc;
                            }
                            const float4* src = land + static_cast<int64_t>(w - w0) * kUnitF4 + frow;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float4 x4 = src[i * kWRows];
                                v[4 * i] += x4.x;
                                v[4 * i + 1] += x4.y;
                                v[4 * i + 2] += x4.z;
                                v[4 * i + 3] += x4.w;
                            }
                        }
                        tmem_st16(acc0 + (cur / nu) * p.acc_stride + (cur % nu) * 16, v);
                        named_bar_sync(1, 128);  // landing buffer free before the next batch
                    }
                                    }
                }
                if (etid == 0) STREAM_TRACE(6);
                // Stage bf16 outputs [token][128 features] in smem, then
                // coalesced 16-byte row stores.
                if (p.rope_tab != nullptr) {
                    // Pull this thread's RoPE table lines toward L1 while the
                    // accumulator is staged: the row-store pass then hits.
                    const int vec = kWRows / 8;
                    for (int v = etid; v < p.M * vec; v += 128) {
                        const float2* tb = p.rope_tab + static_cast<int64_t>(v / vec) * (kWRows / 2) + (v % vec & 7) * 8;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(tb));
                    }
                }
                uint8_t* stage_base = smem + (fused_nq > 0 ? p.stage_off : 0);
                uint16_t* stage = reinterpret_cast<uint16_t*>(stage_base);
                float* stage_f = reinterpret_cast<float*>(stage_base);  // residual: fp32 staging, one rounding after the add
                const float4* land = reinterpret_cast<const float4*>(smem);
                constexpr int kOut = EPI == kSwiGLU ? 1 : NMMA;
                for (int j = 0; j < kOut; ++j) {
                    const int64_t feat0 = static_cast<int64_t>(EPI == kSwiGLU ? t : t * NMMA + j) * kWRows;
                    for (int col = 0; col < cols; col += 16) {
                        float acc[2][16];
#pragma unroll
                        for (int jj = 0; jj < NMMA; ++jj)
                            if (EPI == kSwiGLU || jj == j) {
                                tmem_ld16(acc0 + jj * p.acc_stride + col, acc[jj]);
                                for (int q = 0; q < fused_nq; ++q) {
                                    const float4* src = land + static_cast<int64_t>(q) * slot_f4 +
                                                        (static_cast<int64_t>(jj * nch + (col >> 4)) * 4) * kWRows + frow;
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        const float4 w = src[i * kWRows];
                                        acc[jj][4 * i] += w.x;
                                        acc[jj][4 * i + 1] += w.y;
                                        acc[jj][4 * i + 2] += w.z;
                                        acc[jj][4 * i + 3] += w.w;
                                    }
                                }
                            }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float v = epi_value<EPI>(acc, j, i);
                            if constexpr (EPI == kResidual)
                                stage_f[(col + i) * kWRows + frow] = v;
                            else
                                stage[(col + i) * kWRows + frow] = f2bf(v);
                        }
                    }
                    if (etid == 0) STREAM_TRACE(10);
                    named_bar_sync(1, 128);
                    const int vec = kWRows / 8;  // 16-byte vectors per token row
                    if (EPI != kResidual && p.rope_tab == nullptr) {
                        // Plain rows: four 16-byte vectors per thread in flight
                        // (smem loads first, then the global stores).
                        const int nv = p.M * vec;
                        int v = etid;
                        for (; v + 3 * 128 < nv; v += 4 * 128) {
                            uint4 q[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int vv = v + u * 128;
                                q[u] = *reinterpret_cast<const uint4*>(stage + (vv / vec) * kWRows + (vv % vec) * 8);
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int vv = v + u * 128;
                                *reinterpret_cast<uint4*>(p.c + static_cast<int64_t>(vv / vec) * p.ldc + feat0 + (vv % vec) * 8) = q[u];
                            }
                        }
                        for (; v < nv; v += 128)
                            *reinterpret_cast<uint4*>(p.c + static_cast<int64_t>(v / vec) * p.ldc + feat0 + (v % vec) * 8) =
                                *reinterpret_cast<const uint4*>(stage + (v / vec) * kWRows + (v % vec) * 8);
                    } else
                    for (int v = etid; v < p.M * vec; v += 128) {
                        const int row = v / vec, x = v % vec;
                        uint16_t* o = p.c + static_cast<int64_t>(row) * p.ldc + feat0 + x * 8;
                        if constexpr (EPI == kResidual) {
                            // Residual rows read as 16-byte vectors (coalesced) here
                            // rather than element-wise in the TMEM pass.
                            const uint4 rv = *reinterpret_cast<const uint4*>(p.r + static_cast<int64_t>(row) * p.ldc + feat0 + x * 8);
                            const float4 a = *reinterpret_cast<const float4*>(stage_f + row * kWRows + x * 8);
                            const float4 b = *reinterpret_cast<const float4*>(stage_f + row * kWRows + x * 8 + 4);
                            const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
                            const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                            uint32_t ow[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                ow[e] = pack2(f[2 * e] + bf2f(static_cast<uint16_t>(rw[e] & 0xffffu)),
                                              f[2 * e + 1] + bf2f(static_cast<uint16_t>(rw[e] >> 16)));
                            *reinterpret_cast<uint4*>(o) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                        } else if (p.rope_tab != nullptr) {
                            rope_row_store(p, stage, row, x, static_cast<int>(feat0 / kWRows), o);
                        } else {
                            *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(stage + row * kWRows + x * 8);
                        }
                    }
                    if (etid == 0) STREAM_TRACE(11);
                    named_bar_sync(1, 128);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
        }
    }
    if (threadIdx.x == 64) STREAM_TRACE(7);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) write_end_mark(p.t_end, p.end_cnt);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, p.tmem_cols);
    }
}

// ------------------------------------------------------------ host side ----

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
    bool b_kblocked = false;  // weights in the K-blocked layout (make_map_kblocked)
};

// Weight (B operand) map: a 3D (64, rows, k-blocks) view, one k-block per box.
inline int make_weight_map(CUtensorMap* m, const Launch& L, int box_rows) {
    return L.b_kblocked ? make_map_kblocked(m, L.b, L.b_rows, L.K, box_rows, 1)
                        : make_map_kchunks(m, L.b, L.b_rows, L.K, box_rows, 1);
}

template <int BN, int EPI, bool PAIRED, int STAGES>
int launch(const Launch& L, cudaStream_t stream) {
    using C = Cfg<BN, STAGES>;
    CUtensorMap ma, mb;
    int rc = make_map(&ma, L.a, L.a_rows, L.K, BM);
    if (rc) return rc;
    rc = make_weight_map(&mb, L, PAIRED ? BN / 2 : BN);
    if (rc) return rc;
    static bool configured = false;  // per template instance
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI, PAIRED, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
        configured = true;
    }
    const dim3 grid(L.n_tiles, (L.M + BM - 1) / BM, L.splits);
    if (int rc_ = launch_pdl(gemm_bf16_tcgen05<BN, EPI, PAIRED, STAGES>, dim3(grid), dim3(kThreads), C::kSmemBytes, stream, ma, mb, static_cast<int>(L.row_offset), L.M, L.K / BK / L.splits, L.b_half_rows, L.c, L.ldc, L.r, L.ws,
        L.ws_ld, g_stream_hint)) return rc_;
    return check_launch();
}

int g_persistent = 1;  // kl_tune(KL_TUNE_GEMM_PERSISTENT, ...)
int sm_count();

template <int BN, int EPI, bool PAIRED, int STAGES>
int launch_persistent(const Launch& L, cudaStream_t stream) {
    using C = Cfg<BN, STAGES>;
    CUtensorMap ma, mb;
    int rc = make_map(&ma, L.a, L.a_rows, L.K, BM);
    if (rc) return rc;
    rc = make_weight_map(&mb, L, PAIRED ? BN / 2 : BN);
    if (rc) return rc;
    static bool configured = false;
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_persistent_tcgen05<BN, EPI, PAIRED, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes + 64));
        configured = true;
    }
    const int m_tiles = (L.M + BM - 1) / BM;
    const int total = L.n_tiles * m_tiles;
    const int grid = std::min(total, sm_count());
    gemm_persistent_tcgen05<BN, EPI, PAIRED, STAGES><<<grid, kThreads, C::kSmemBytes + 64, stream>>>(
        ma, mb, static_cast<int>(L.row_offset), L.M, L.K / BK, L.b_half_rows, L.n_tiles, m_tiles, L.c, L.ldc, L.r);
    return check_launch();
}

template <int EPI>
int reduce(const Launch& L, int n_out, int pair_bn, cudaStream_t stream) {
    const int64_t threads = static_cast<int64_t>(L.M) * (n_out / 4);
    if (int rc_ = launch_pdl(splitk_reduce_kernel<EPI>, dim3(static_cast<int>((threads + 255) / 256)), dim3(256), 0, stream, L.ws, L.splits, L.M, L.ws_ld, n_out, pair_bn, L.c, L.ldc, L.r)) return rc_;
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

// --- weight-streaming path (host) ---
int g_stream_enabled = 1;  // kl_tune(KL_TUNE_STREAM_GEMM, ...)
int g_stream_nmma = 1;     // kl_tune(KL_TUNE_STREAM_NMMA, ...): weight sub-tiles per activation tile
int g_stream_stages = 8;   // kl_tune(KL_TUNE_STREAM_STAGES, ...): cap on the smem ring depth
int g_stream_ctas = 1;     // kl_tune(KL_TUNE_STREAM_CTAS_PER_SM, ...)
int g_stream_debug = 0;
int g_stream_whole_tiles = 70;  // kl_tune(KL_TUNE_STREAM_WHOLE_TILES, pct): whole tiles when n_tiles >= pct% of SMs
int g_stream_even_split = 2;  // kl_tune(KL_TUNE_STREAM_EVEN_SPLIT, ...): 1 = equal splits only, 2 (default) = also near-equal
int g_stream_fused_fixup = 1;  // kl_tune(KL_TUNE_STREAM_FUSED_FIXUP, 0|1)
int g_stream_ks = 3;  // kl_tune(KL_TUNE_STREAM_KBLOCKS_PER_STAGE, 1|2|3): 2 k-blocks per stage where >= 3 (2) or >= 2 (3) stages fit

int sm_count() {
    static const int n = [] {
        int dev = 0, v = kSMs;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            return v;
        cudaGetLastError();
        return kSMs;
    }();
    return n;
}

uint32_t next_epoch() {
    static std::atomic<uint32_t> e{0};
    uint32_t v = ++e;
    while (v == 0) v = ++e;
    return v;
}

constexpr int64_t kFlagBytes = 1024;  // [<= 256 CTAs] uint32 publish epochs
constexpr int kStreamSmemBudget = 227 * 1024 - 2048;  // + 1 KB alignment + 1 KB barriers

int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}
int stream_np(int M) { return std::max(16, (M + 15) & ~15); }
bool stream_eligible(int M, int N, int K, int epilogue) {
    if (!g_stream_enabled || M < 1 || M > 256) return false;
    if (!(epilogue == kSwiGLU ? (N / 2) % kWRows == 0 : N % kWRows == 0)) return false;
    // Below ~40 MB of weights the persistent kernel's ramp and split fixup
    // outweigh its balance; the one-tile-per-CTA kernel wins there unless
    // the rows need two of its 128-row tiles (each re-reading the weights).
    return M > 128 || static_cast<int64_t>(N) * K * 2 >= (40LL << 20) || g_stream_enabled == 2;
}
int stream_nmma(int N, int epilogue) {
    if (epilogue == kSwiGLU) return 2;
    return (g_stream_nmma == 2 && N % (2 * kWRows) == 0) ? 2 : 1;
}
int64_t stream_slot_bytes(int M, int nmma) { return static_cast<int64_t>(nmma) * kWRows * stream_np(M) * 4; }
// Persistent grid: one CTA per SM (x g_stream_ctas), at least 4 k-blocks each.
int stream_grid(int N, int K, int epilogue) {
    const int nmma = stream_nmma(N, epilogue);
    const int n_tiles = epilogue == kSwiGLU ? N / 2 / kWRows : N / (kWRows * nmma);
    const int units = n_tiles * (K / BK);
    return std::max(1, std::min(sm_count() * g_stream_ctas, units / 4));
}

struct RopeArgs {
    const float2* table;
    const int32_t* pos;
    const int32_t* seq;
    uint16_t* kc;
    uint16_t* vc;
    int Hq, Hkv, cap, sink, chunk_last_pos;
};

template <int EPI, int NMMA, bool Q4 = false>
int launch_stream(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int64_t b_rows,
                  int n_tiles, int half_rows, uint16_t* c, int ldc, const uint16_t* r, void* ws, int64_t ws_bytes,
                  cudaStream_t stream, const uint8_t* q4 = nullptr, bool wkb = false, const RopeArgs* rope = nullptr,
                  float* defer = nullptr, int64_t defer_split_elems = 0, int defer_splits = 0,
                  EndMark end = EndMark{nullptr, nullptr}) {
    StreamArgs p{};
    p.t_end = end.t;
    p.end_cnt = end.cnt;
    p.defer = defer;
    p.defer_split_elems = defer_split_elems;
    p.defer_ld = static_cast<int>(n_tiles) * kWRows * NMMA;
    if (rope != nullptr) {
        p.rope_tab = rope->table;
        p.rope_pos = rope->pos;
        p.rope_seq = rope->seq;
        p.kc = rope->kc;
        p.vc = rope->vc;
        p.Hq = rope->Hq;
        p.Hkv = rope->Hkv;
        p.cap = rope->cap;
        p.sink = rope->sink;
        p.chunk_last_pos = rope->chunk_last_pos;
    }
    p.M = M;
    p.NP = stream_np(M);
    p.acc_stride = pow2ceil(std::max(32, p.NP));
    p.nbuf = 2 * NMMA * p.acc_stride <= 512 ? 2 : 1;
    p.tmem_cols = static_cast<uint32_t>(std::max(32, p.nbuf * NMMA * p.acc_stride));
    // Two k-blocks per stage (one 3D TMA box each for weights and
    // activations) when K allows: 32-64 KB copies stream HBM faster than
    // 16 KB ones (tools/bw_probe.cu).
    {
        const int per_kb = NMMA * kWTileBytes + p.NP * BK * 2;
        // Knob 3 (default): two k-blocks per stage down to 2 stages. The
        // SwiGLU pair at M = 64..192 (2 x 96 KB stages) streams 2-3 us
        // faster than with 3-5 single-k-block stages (tools/dev/swiglu_probe2.sh).
        const int min_stages = g_stream_ks == 3 ? 2 : 3;
        p.ks = (!Q4 && g_stream_ks >= 2 && (K / BK) % 2 == 0 &&
                std::min(g_stream_stages, kStreamSmemBudget / g_stream_ctas / (2 * per_kb)) >= min_stages)
                   ? 2
                   : 1;  // keep >= 3 stages in flight (the SwiGLU pair's 96 KB stages would leave 2)
    }
    p.KB = K / BK / p.ks;
    p.units = n_tiles * p.KB;
    const int stage_bytes = p.ks * (NMMA * kWTileBytes + p.NP * BK * 2);
    const int per_stage = stage_bytes + (Q4 ? NMMA * kQ4Chunk : 0);
    p.stages = std::min(g_stream_stages, kStreamSmemBudget / g_stream_ctas / per_stage);
    if (p.stages < 2 || p.tmem_cols * g_stream_ctas > 512) return KL_EUNSUPPORTED;
    // The idle ring doubles as the landing buffer of split partials (8 KB
    // units) and as the bf16 output staging tile of the last segment.
    if (p.stages * stage_bytes < p.NP * kWRows * (EPI == kResidual ? 4 : 2)) return KL_EUNSUPPORTED;
    p.hint = g_stream_hint;
    p.debug = g_stream_debug;
    p.pdl = g_pdl;
    if (p.stages > 16) p.stages = 16;
    int G = std::max(1, std::min(sm_count() * g_stream_ctas, p.units / 4));
    if (g_stream_whole_tiles > 0 && n_tiles <= sm_count() && n_tiles * 100 >= g_stream_whole_tiles * sm_count())
        G = n_tiles;  // one whole tile per CTA: no split partials, the rest of the SMs idle
    else if (g_stream_even_split && n_tiles < G && G / n_tiles >= 2 &&
             (p.KB % (G / n_tiles) == 0 || g_stream_even_split == 2 || defer != nullptr)) {
        // Every tile split into the same number S of k-ranges cut at tile
        // boundaries (unit_begin), equal when S divides KB (else the owner's
        // range takes the remainder), the owner's optionally longer.
        G = n_tiles * (G / n_tiles);
        p.split = G / n_tiles;
    }
    if (defer != nullptr) {
        // Deferred splits need exactly the tile-aligned split count the
        // caller sized its partial buffer for; no workspace slots are used.
        if (EPI != kStore || NMMA != 1 || Q4 || p.split != defer_splits) return KL_EUNSUPPORTED;
    }
    const int G_ws = defer != nullptr ? G
                                      : static_cast<int>(std::min<int64_t>(
                                            (ws_bytes - kFlagBytes) / stream_slot_bytes(M, NMMA), kFlagBytes / 4));
    if (G > G_ws) {  // workspace-limited: plain stream-K ranges over fewer CTAs
        G = G_ws;
        p.split = 0;
    }
    if (G < 1) return KL_EUNSUPPORTED;
    // The fused RoPE epilogue runs only on owners' staged path: no CTA range
    // may contain a whole tile strictly inside it.
    if (rope != nullptr && p.split == 0 && (p.units + G - 1) / G > p.KB + 1) return KL_EUNSUPPORTED;
    p.half_rows = half_rows;
    p.c = c;
    p.ldc = ldc;
    p.r = r;
    p.flags = static_cast<uint32_t*>(ws);
    p.ws = reinterpret_cast<float*>(static_cast<char*>(ws) + kFlagBytes);
    p.epoch = next_epoch();
    p.q4 = q4;
    CUtensorMap mw, mx;
    int rc = p.ks > 1 ? make_map_kchunks(&mx, a, a_rows, K, p.NP, p.ks) : make_map(&mx, a, a_rows, K, p.NP);
    if (rc) return rc;
    if (Q4)
        mw = mx;  // unused: the Q4 variant bulk-copies packed tiles
    else if ((rc = wkb ? make_map_kblocked(&mw, b, b_rows, K, kWRows, p.ks) : make_map_kchunks(&mw, b, b_rows, K, kWRows, p.ks)))
        return rc;
    int smem = p.stages * per_stage + 1024 + 1024;  // rings + alignment + barriers
    // A dedicated output staging region after the barriers when it fits:
    // the owner then adds the landed partials during its epilogue pass.
    {
        const int stage_bytes = p.NP * kWRows * (EPI == kResidual ? 4 : 2);
        if (g_stream_fused_fixup && smem + stage_bytes <= kStreamSmemBudget + 2048) {
            p.stage_off = p.stages * per_stage + 1024;
            smem += stage_bytes;
        }
    }
    static bool configured = false;  // per template instance
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_stream_kernel<EPI, NMMA, Q4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kStreamSmemBudget + 2048));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kStreamThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl ? 1 : 0;
    p.t_start = t_next_start;
    t_next_start = nullptr;
    KL_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_stream_kernel<EPI, NMMA, Q4>, mw, mx, static_cast<int>(row_offset), p));
    return check_launch();
}

int gemm_stream(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int N,
                uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* ws, int64_t ws_bytes, cudaStream_t stream,
                bool wkb) {
    const int nmma = stream_nmma(N, epilogue);
    if (epilogue == kSwiGLU)
        return launch_stream<kSwiGLU, 2>(a, a_rows, row_offset, M, K, b, N, N / 2 / kWRows, N / 2, c, ldc, r, ws,
                                         ws_bytes, stream, nullptr, wkb);
    const int n_tiles = N / (kWRows * nmma);
    if (epilogue == kResidual)
        return nmma == 2 ? launch_stream<kResidual, 2>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws,
                                                       ws_bytes, stream, nullptr, wkb)
                         : launch_stream<kResidual, 1>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws,
                                                       ws_bytes, stream, nullptr, wkb);
    return nmma == 2 ? launch_stream<kStore, 2>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws, ws_bytes,
                                                stream, nullptr, wkb)
                     : launch_stream<kStore, 1>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws, ws_bytes,
                                                stream, nullptr, wkb);
}

}  // namespace
}  // namespace kl

extern "C" int kl_stamp_next_launch(unsigned long long* dst) {
    kl::t_next_start = dst;
    return KL_OK;
}

extern "C" int kl_stream_trace(unsigned long long* host, int n_ctas) {
    const int rc = static_cast<int>(cudaMemcpyFromSymbol(host, kl::g_stream_trace, static_cast<size_t>(n_ctas) * 12 * 8));
    static unsigned long long zero[256 * 12] = {};
    cudaMemcpyToSymbol(kl::g_stream_trace, zero, sizeof(zero));
    return rc;
}

namespace kl {
extern int g_prefill_tc;
extern int g_decode_mma;
extern int g_decode_hg;
extern int g_attn_kv_evict_first;
extern int g_decode_stages;
extern int g_rope_tok;
}

extern "C" int kl_tune(int knob, int value) {
    using namespace kl;
    switch (knob) {
        case KL_TUNE_STREAM_GEMM: g_stream_enabled = value; return KL_OK;
        case KL_TUNE_STREAM_NMMA:
            if (value != 1 && value != 2) return KL_EINVAL;
            g_stream_nmma = value;
            return KL_OK;
        case KL_TUNE_STREAM_STAGES:
            if (value < 2 || value > 16) return KL_EINVAL;
            g_stream_stages = value;
            return KL_OK;
        case KL_TUNE_STREAM_HINT: g_stream_hint = value; return KL_OK;
        case 99: g_stream_debug = value; return KL_OK;
        case KL_TUNE_PDL: g_pdl = value != 0; return KL_OK;
        case KL_TUNE_PREFILL_TC: g_prefill_tc = value; return KL_OK;
        case KL_TUNE_DECODE_MMA: g_decode_mma = value; return KL_OK;
        case KL_TUNE_DECODE_HG: g_decode_hg = value < 0 ? 0 : value; return KL_OK;
        case KL_TUNE_ATTN_KV_EVICT_FIRST: g_attn_kv_evict_first = value != 0; return KL_OK;
        case KL_TUNE_DECODE_STAGES: g_decode_stages = value < 0 || value > 12 ? 0 : value; return KL_OK;
        case KL_TUNE_ROPE_TOKEN_BLOCKS: g_rope_tok = value != 0; return KL_OK;
        case KL_TUNE_STREAM_WHOLE_TILES: g_stream_whole_tiles = value; return KL_OK;
        case KL_TUNE_GEMM_PERSISTENT: g_persistent = value != 0; return KL_OK;
        case KL_TUNE_STREAM_EVEN_SPLIT: g_stream_even_split = value; return KL_OK;
        case KL_TUNE_STREAM_FUSED_FIXUP: g_stream_fused_fixup = value != 0; return KL_OK;
        case KL_TUNE_STREAM_KBLOCKS_PER_STAGE:
            if (value < 1 || value > 3) return KL_EINVAL;
            g_stream_ks = value;
            return KL_OK;
        case KL_TUNE_STREAM_CTAS_PER_SM:
            if (value != 1 && value != 2) return KL_EINVAL;
            g_stream_ctas = value;
            return KL_OK;
        default: return KL_EINVAL;
    }
}

extern "C" int64_t kl_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
    using namespace kl;
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    if (stream_eligible(M, N, K, epilogue))
        return kFlagBytes + static_cast<int64_t>(stream_grid(N, K, epilogue)) * stream_slot_bytes(M, stream_nmma(N, epilogue));
    const int m_tiles = (M + BM - 1) / BM;
    const int tiles = (N / 128) * m_tiles;
    const int s = choose_splits(tiles, K / BK, M, N, INT64_MAX);
    (void)epilogue;
    return s > 1 ? static_cast<int64_t>(s) * M * N * 4 : 0;
}

namespace kl {
namespace {
// kl_gemm_bf16 / kl_gemm_bf16_kb: b row-major [N, K] or K-blocked (wkb).
int gemm_bf16_impl(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int N,
                   uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace, int64_t workspace_bytes,
                   cudaStream_t stream, bool wkb) {
    if (M < 0 || K <= 0 || N <= 0 || a == nullptr || b == nullptr || c == nullptr) return KL_EINVAL;
    if (M == 0) return KL_OK;
    if (K % BK != 0 || N % 64 != 0 || !aligned16(a) || !aligned16(b) || !aligned16(c) || ldc % 8 != 0)
        return KL_EINVAL;
    if (row_offset < 0 || row_offset + M > a_rows || row_offset > INT32_MAX) return KL_EINVAL;
    if (epilogue < 0 || epilogue > 2) return KL_EINVAL;
    if (epilogue == kResidual && (r == nullptr || !aligned16(r))) return KL_EINVAL;
    if (epilogue == kSwiGLU && N % 256 != 0) return KL_EINVAL;
    if (workspace != nullptr && !aligned16(workspace)) return KL_EINVAL;
    if (workspace != nullptr && stream_eligible(M, N, K, epilogue) &&
        workspace_bytes >= kFlagBytes + stream_slot_bytes(M, stream_nmma(N, epilogue))) {
        const int rc = gemm_stream(a, a_rows, row_offset, M, K, b, N, c, ldc, r, epilogue, workspace, workspace_bytes,
                                   stream, wkb);
        if (rc != KL_EUNSUPPORTED) return rc;
    }
    if (t_next_start != nullptr) {  // a pending op-start mark on a non-streaming path: a separate stamp
        unsigned long long* ts = t_next_start;
        t_next_start = nullptr;
        if (const int rc = kl_stamp(ts, stream)) return rc;
    }
    const int m_tiles = (M + BM - 1) / BM;
    const int kb = K / BK;
    Launch L{a, a_rows, row_offset, M, K, b, N, 0, 0, c, ldc, r, 1, static_cast<float*>(workspace), N, wkb};
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
    // Compute-bound regime (prefill / large M): 256-wide tiles, deep pipeline;
    // persistent with double-buffered accumulators once there are more tiles
    // than SMs.
    const bool persist = g_persistent && static_cast<int64_t>(N / 256) * m_tiles > sm_count();
    if (epilogue == kSwiGLU) {
        L.n_tiles = N / 256;
        L.b_half_rows = N / 2;
        return persist ? launch_persistent<256, kSwiGLU, true, 4>(L, stream) : launch<256, kSwiGLU, true, 4>(L, stream);
    }
    if (N % 256 == 0) {
        L.n_tiles = N / 256;
        if (persist)
            return epilogue == kResidual ? launch_persistent<256, kResidual, false, 4>(L, stream)
                                         : launch_persistent<256, kStore, false, 4>(L, stream);
        return epilogue == kResidual ? launch<256, kResidual, false, 4>(L, stream)
                                     : launch<256, kStore, false, 4>(L, stream);
    }
    L.n_tiles = N / 64;
    return epilogue == kResidual ? launch<64, kResidual, false, 6>(L, stream) : launch<64, kStore, false, 6>(L, stream);
}
}  // namespace
}  // namespace kl

extern "C" int kl_gemm_bf16(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b,
                            int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace,
                            int64_t workspace_bytes, cudaStream_t stream) {
    return kl::gemm_bf16_impl(a, a_rows, row_offset, M, K, b, N, c, ldc, r, epilogue, workspace, workspace_bytes, stream,
                              false);
}

extern "C" int kl_gemm_bf16_kb(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b,
                               int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace,
                               int64_t workspace_bytes, cudaStream_t stream) {
    return kl::gemm_bf16_impl(a, a_rows, row_offset, M, K, b, N, c, ldc, r, epilogue, workspace, workspace_bytes, stream,
                              true);
}

extern "C" int kl_gemm_bf16_qkv_rope(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                                     const uint16_t* b, int Hq, int Hkv, int hd, uint16_t* c, int ldc,
                                     const float* rope_table, const int32_t* pos, const int32_t* seq, uint16_t* k_cache,
                                     uint16_t* v_cache, int cap, int sink, int chunk_last_pos, void* workspace,
                                     int64_t workspace_bytes, cudaStream_t stream) {
    using namespace kl;
    if (M < 0 || K <= 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || !a || !b || !c || !rope_table || !pos || !seq || !k_cache ||
        !v_cache || cap <= sink || sink < 0)
        return KL_EINVAL;
    if (M == 0) return KL_OK;
    const int N = (Hq + 2 * Hkv) * hd;
    // One 128-row weight tile per head, on the weight-streaming path.
    if (hd != kWRows || K % BK != 0 || !aligned16(a) || !aligned16(b) || !aligned16(c) || ldc % 8 != 0 ||
        !aligned16(k_cache) || !aligned16(v_cache) || row_offset < 0 || row_offset + M > a_rows)
        return KL_EUNSUPPORTED;
    if (workspace == nullptr || !aligned16(workspace) || !stream_eligible(M, N, K, kStore) ||
        workspace_bytes < kFlagBytes + stream_slot_bytes(M, 1))
        return KL_EUNSUPPORTED;
    const RopeArgs ra{reinterpret_cast<const float2*>(rope_table), pos, seq, k_cache, v_cache, Hq, Hkv, cap, sink,
                      chunk_last_pos};
    return launch_stream<kStore, 1>(a, a_rows, row_offset, M, K, b, N, N / kWRows, 0, c, ldc, nullptr, workspace,
                                    workspace_bytes, stream, nullptr, false, &ra);
}

extern "C" int kl_gemm_q4(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint8_t* bq,
                          int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace,
                          int64_t workspace_bytes, cudaStream_t stream) {
    using namespace kl;
    if (M < 0 || K <= 0 || N <= 0 || a == nullptr || bq == nullptr || c == nullptr) return KL_EINVAL;
    if (M == 0) return KL_OK;
    if (M > 256) return KL_EUNSUPPORTED;  // large M: kl_dequantize_q4 + kl_gemm_bf16
    if (K % BK != 0 || N % kWRows != 0 || (epilogue == kSwiGLU && (N / 2) % kWRows != 0) || ldc % 8 != 0)
        return KL_EINVAL;
    if (epilogue < 0 || epilogue > 2 || (epilogue == kResidual && r == nullptr)) return KL_EINVAL;
    if (row_offset < 0 || row_offset + M > a_rows || workspace == nullptr ||
        workspace_bytes < kFlagBytes + stream_slot_bytes(M, epilogue == kSwiGLU ? 2 : 1))
        return KL_EINVAL;
    // NMMA = 1 for plain GEMMs (fewest split contributors), the gate/up pair for SwiGLU.
    if (epilogue == kSwiGLU)
        return launch_stream<kSwiGLU, 2, true>(a, a_rows, row_offset, M, K, nullptr, N, N / 2 / kWRows, N / 2, c, ldc,
                                               r, workspace, workspace_bytes, stream, bq);
    if (epilogue == kResidual)
        return launch_stream<kResidual, 1, true>(a, a_rows, row_offset, M, K, nullptr, N, N / kWRows, 0, c, ldc, r,
                                                 workspace, workspace_bytes, stream, bq);
    return launch_stream<kStore, 1, true>(a, a_rows, row_offset, M, K, nullptr, N, N / kWRows, 0, c, ldc, r, workspace,
                                          workspace_bytes, stream, bq);
}

extern "C" int64_t kl_gemm_q4_workspace_bytes(int M, int N, int K, int epilogue) {
    using namespace kl;
    if (M <= 0 || M > 256 || N <= 0 || K <= 0) return 0;
    const int nmma = epilogue == kSwiGLU ? 2 : 1;
    const int n_tiles = epilogue == kSwiGLU ? N / 2 / kWRows : N / kWRows;
    const int G = std::max(1, std::min(sm_count(), n_tiles * (K / BK) / 4));
    return kFlagBytes + static_cast<int64_t>(G) * stream_slot_bytes(M, nmma);
}

extern "C" int kl_expert_ffn_q4(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d, int f,
                                const uint8_t* w13q, const uint8_t* w2q, uint16_t* h_scratch, uint16_t* y,
                                void* workspace, int64_t workspace_bytes, cudaStream_t stream) {
    if (M == 0) return KL_OK;
    if (y == nullptr || h_scratch == nullptr) return KL_EINVAL;
    int rc = kl_gemm_q4(xp, rows_total, row_offset, M, d, w13q, 2 * f, h_scratch, f, nullptr, 2, workspace,
                        workspace_bytes, stream);
    if (rc) return rc;
    return kl_gemm_q4(h_scratch, M, 0, M, f, w2q, d, y + row_offset * d, d, nullptr, 0, workspace, workspace_bytes,
                      stream);
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

extern "C" int kl_expert_ffn_kb(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d, int f,
                                const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch, uint16_t* y,
                                void* workspace, int64_t workspace_bytes, cudaStream_t stream) {
    if (M == 0) return KL_OK;
    if (y == nullptr || h_scratch == nullptr) return KL_EINVAL;
    int rc = kl_gemm_bf16_kb(xp, rows_total, row_offset, M, d, w13, 2 * f, h_scratch, f, nullptr, 2, workspace,
                             workspace_bytes, stream);
    if (rc) return rc;
    return kl_gemm_bf16_kb(h_scratch, M, 0, M, f, w2, d, y + row_offset * d, d, nullptr, 0, workspace, workspace_bytes,
                           stream);
}

// Tile-aligned split count launch_stream picks for a deferred [N, K]
// weight-streaming GEMM at M rows (near-equal splits allowed), 0 when that
// GEMM would not run as tile-aligned splits (or S > 4).
extern "C" int kl_gemm_deferred_splits(int M, int N, int K) {
    using namespace kl;
    // No size threshold here: the small-GEMM reason to avoid the streaming
    // kernel (its split fixup tail) does not exist when splits are deferred.
    if (M < 1 || M > 256 || N % kWRows != 0 || K % BK != 0 || !g_stream_enabled) return 0;
    if (stream_nmma(N, kStore) != 1) return 0;
    const int NP = stream_np(M);
    const int per_kb = kWTileBytes + NP * BK * 2;
    const int min_stages = g_stream_ks == 3 ? 2 : 3;
    const int ks = (g_stream_ks >= 2 && (K / BK) % 2 == 0 &&
                    std::min(g_stream_stages, kStreamSmemBudget / g_stream_ctas / (2 * per_kb)) >= min_stages)
                       ? 2
                       : 1;
    const int KB = K / BK / ks, n_tiles = N / kWRows;
    const int G = std::max(1, std::min(sm_count() * g_stream_ctas, n_tiles * KB / 4));
    if (g_stream_whole_tiles > 0 && n_tiles <= sm_count() && n_tiles * 100 >= g_stream_whole_tiles * sm_count())
        return 0;
    if (!(g_stream_even_split && n_tiles < G && G / n_tiles >= 2)) return 0;
    const int S = G / n_tiles;
    return S <= 4 ? S : 0;
}

// The down projection defers only where the owner-fixup form would also run
// on the streaming kernel (>= 40 MB of weights or M > 128), so a deferred and
// a non-deferred FFN (e.g. an expert-parallel shard) share split partitions.
extern "C" int kl_expert_ffn_deferred_splits(int M, int d, int f) {
    return kl::stream_eligible(M, d, f, kl::kStore) ? kl_gemm_deferred_splits(M, d, f) : 0;
}

extern "C" int kl_gemm_bf16_deferred(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                                     const uint16_t* b, int N, int b_kblocked, float* c_part, int64_t part_rows,
                                     int splits, void* workspace, int64_t workspace_bytes, cudaStream_t stream) {
    using namespace kl;
    if (M == 0) return KL_OK;
    if (c_part == nullptr || a == nullptr || b == nullptr || splits < 2 || splits > 4 || M > part_rows ||
        row_offset < 0 || row_offset + M > a_rows || !aligned16(a) || !aligned16(b))
        return KL_EINVAL;
    if (kl_gemm_deferred_splits(M, N, K) != splits) return KL_EUNSUPPORTED;
    return launch_stream<kStore, 1>(a, a_rows, row_offset, M, K, b, N, N / kWRows, 0, nullptr, N, nullptr, workspace,
                                    workspace_bytes, stream, nullptr, b_kblocked != 0, nullptr, c_part,
                                    part_rows * N, splits, take_next_end());
}

extern "C" int kl_expert_ffn_kb_deferred(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d,
                                         int f, const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch,
                                         float* y_part, int64_t part_rows, int splits, void* workspace,
                                         int64_t workspace_bytes, cudaStream_t stream) {
    using namespace kl;
    if (M == 0) return KL_OK;
    if (y_part == nullptr || h_scratch == nullptr || splits < 2 || splits > 4 || row_offset < 0 ||
        row_offset + M > part_rows || !aligned16(h_scratch) || !aligned16(w2))
        return KL_EINVAL;
    if (kl_expert_ffn_deferred_splits(M, d, f) != splits) return KL_EUNSUPPORTED;
    int rc = kl_gemm_bf16_kb(xp, rows_total, row_offset, M, d, w13, 2 * f, h_scratch, f, nullptr, 2, workspace,
                             workspace_bytes, stream);
    if (rc) return rc;
    return launch_stream<kStore, 1>(h_scratch, M, 0, M, f, w2, d, d / kWRows, 0, nullptr, d, nullptr, workspace,
                                    workspace_bytes, stream, nullptr, true, nullptr, y_part + row_offset * d,
                                    part_rows * d, splits, take_next_end());
}

namespace kl {
namespace {
// Row-major [rows, cols] -> K-blocked (cols/64 slabs of [rows][64]); one
// 16-byte vector per thread.
__global__ void kblock_kernel(const uint4* __restrict__ src, int64_t rows, int64_t cols, uint4* __restrict__ dst) {
    const int64_t n16 = rows * cols / 8;
    const int64_t cpr = cols / 8;  // 16-byte vectors per source row
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = i / cpr, v = i % cpr;  // v: 16-byte vector within the row
        const int64_t slab = v / 8, within = v % 8;
        dst[(slab * rows + row) * 8 + within] = src[i];
    }
}
}  // namespace
}  // namespace kl

extern "C" int kl_weights_kblock(const uint16_t* src, int64_t rows, int64_t cols, uint16_t* dst, cudaStream_t stream) {
    using namespace kl;
    if (src == nullptr || dst == nullptr || rows <= 0 || cols <= 0 || cols % 64 != 0 || src == dst) return KL_EINVAL;
    if (!aligned16(src) || !aligned16(dst)) return KL_EINVAL;
    const int64_t n16 = rows * cols / 8;
    const int grid = static_cast<int>(std::min<int64_t>((n16 + 255) / 256, 148LL * 16));
    kblock_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const uint4*>(src), rows, cols, reinterpret_cast<uint4*>(dst));
    return check_launch();
}
