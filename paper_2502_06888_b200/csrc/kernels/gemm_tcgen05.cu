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
    int KB;         // k-blocks per tile
    int units;      // n_tiles * KB
    int half_rows;  // SwiGLU: first W3 row inside B
    int stages;
    uint16_t* c;
    int ldc;
    const uint16_t* r;
    float* ws;        // [grid][NMMA][128][NP] fp32 partial slots
    uint32_t* flags;  // [grid] publish epochs
    uint32_t epoch;
    uint32_t tmem_cols;
};

__device__ __forceinline__ int range_begin(int c, int units, int G) {
    return static_cast<int>(static_cast<int64_t>(c) * units / G);
}

template <int EPI, int NMMA>
__global__ void __launch_bounds__(kStreamThreads, 1)
gemm_stream_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, int a_row0,
                   const StreamArgs p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = NMMA * kWTileBytes + p.NP * BK * 2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty = full + p.stages;
    uint64_t* acc_full = empty + p.stages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, cta = blockIdx.x;
    const int KB = p.KB;
    const int u0 = range_begin(cta, p.units, G), u1 = range_begin(cta + 1, p.units, G);
    const int t_hi = u1 > u0 ? (u1 - 1) / KB : 0, t_lo = u1 > u0 ? u0 / KB : 1;  // tiles walked t_hi .. t_lo

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_x = l2_policy_evict_last();
            int it = 0;
            for (int t = t_hi; t >= t_lo; --t) {
                const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % p.stages;
                    mbar_wait(&empty[s], ((it / p.stages) & 1) ^ 1);
                    uint8_t* sw = smem + s * stage_bytes;
                    mbar_arrive_expect_tx(&full[s], stage_bytes);
#pragma unroll
                    for (int j = 0; j < NMMA; ++j) {
                        const int row = EPI == kSwiGLU ? (j == 0 ? t * kWRows : p.half_rows + t * kWRows)
                                                       : (t * NMMA + j) * kWRows;
                        tma_load_2d_hint(sw + j * kWTileBytes, &tmap_w, &full[s], kb * BK, row, pol_w);
                    }
                    tma_load_2d_hint(sw + NMMA * kWTileBytes, &tmap_x, &full[s], kb * BK, a_row0, pol_x);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16_f32(kWRows, p.NP);
            int it = 0, seg = 0;
            for (int t = t_hi; t >= t_lo; --t, ++seg) {
                const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
                mbar_wait(acc_empty, (seg & 1) ^ 1);  // epilogue drained the previous segment
                tc_fence_after();
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % p.stages;
                    mbar_wait(&full[s], (it / p.stages) & 1);
                    tc_fence_after();
                    const uint32_t sw = smem_u32(smem + s * stage_bytes);
                    const uint32_t sx = sw + NMMA * kWTileBytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
#pragma unroll
                        for (int j = 0; j < NMMA; ++j)
                            tc_mma_bf16(tmem_base + j * p.acc_stride, sw128_kmajor_desc(sw + j * kWTileBytes + k * 32),
                                        sw128_kmajor_desc(sx + k * 32), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    tc_commit(&empty[s]);
                }
                tc_commit(acc_full);
            }
        }
        __syncwarp();
    } else {
        const int quarter = warp & 3;
        const int frow = quarter * 32 + lane;  // feature row inside a 128-row sub-tile
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
        const int cols = (p.M + 15) & ~15;  // token columns worth reading
        int seg = 0;
        for (int t = t_hi; t >= t_lo; --t, ++seg) {
            const int kb0 = max(u0, t * KB) - t * KB, kb1 = min(u1, (t + 1) * KB) - t * KB;
            mbar_wait(acc_full, seg & 1);
            tc_fence_after();
            const bool has_last = kb1 == KB;
            if (!has_last) {
                // Contributor: publish the fp32 partial of this tile.
                float* slot = p.ws + static_cast<int64_t>(cta) * NMMA * kWRows * p.NP;
                for (int j = 0; j < NMMA; ++j) {
                    float* dst = slot + (static_cast<int64_t>(j) * kWRows + frow) * p.NP;
                    for (int col = 0; col < cols; col += 16) {
                        float v[16];
                        tmem_ld16(lane_addr + j * p.acc_stride + col, v);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            __stcg(reinterpret_cast<float4*>(dst + col) + i,
                                   make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
                    }
                }
                __threadfence();
                named_bar_sync(1, 128);
                if (warp == 2 && lane == 0) st_release_gpu(p.flags + cta, p.epoch);
            } else {
                // Full tile, or owner of a split tile: contributors are the
                // CTAs c_lo .. cta-1 holding k-blocks [t*KB, u0).
                int c_lo = cta;
                if (kb0 > 0) {
                    c_lo = cta - 1;
                    while (c_lo > 0 && range_begin(c_lo, p.units, G) > t * KB) --c_lo;
                    for (int q = c_lo; q < cta; ++q)
                        while (ld_acquire_gpu(p.flags + q) != p.epoch) {
                        }
                }
                for (int col = 0; col < cols; col += 16) {
                    float acc[NMMA][16];
#pragma unroll
                    for (int j = 0; j < NMMA; ++j) tmem_ld16(lane_addr + j * p.acc_stride + col, acc[j]);
                    for (int q = c_lo; q < cta; ++q) {
                        const float* slot = p.ws + static_cast<int64_t>(q) * NMMA * kWRows * p.NP;
#pragma unroll
                        for (int j = 0; j < NMMA; ++j) {
                            const float4* src =
                                reinterpret_cast<const float4*>(slot + (static_cast<int64_t>(j) * kWRows + frow) * p.NP + col);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float4 w = __ldcg(src + i);
                                acc[j][4 * i] += w.x;
                                acc[j][4 * i + 1] += w.y;
                                acc[j][4 * i + 2] += w.z;
                                acc[j][4 * i + 3] += w.w;
                            }
                        }
                    }
                    if constexpr (EPI == kSwiGLU) {
                        uint16_t* out = p.c + static_cast<int64_t>(col) * p.ldc + t * kWRows + frow;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            if (col + i < p.M) {
                                const float g = acc[0][i], u = acc[1][i];
                                out[static_cast<int64_t>(i) * p.ldc] = f2bf(g / (1.0f + expf(-g)) * u);
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NMMA; ++j) {
                            const int64_t feat = static_cast<int64_t>(t * NMMA + j) * kWRows + frow;
                            uint16_t* out = p.c + static_cast<int64_t>(col) * p.ldc + feat;
                            const uint16_t* res = EPI == kResidual ? p.r + static_cast<int64_t>(col) * p.ldc + feat : nullptr;
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                if (col + i < p.M) {
                                    float v = acc[j][i];
                                    if constexpr (EPI == kResidual) v += bf2f(res[static_cast<int64_t>(i) * p.ldc]);
                                    out[static_cast<int64_t>(i) * p.ldc] = f2bf(v);
                                }
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, p.tmem_cols);
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

// --- weight-streaming path (host) ---
int g_stream_enabled = 1;  // kl_tune(KL_TUNE_STREAM_GEMM, ...)
int g_stream_nmma = 2;     // kl_tune(KL_TUNE_STREAM_NMMA, ...): weight sub-tiles per activation tile

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
constexpr int kStreamSmemBudget = 227 * 1024 - 1024 - 256;

int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}
int stream_np(int M) { return std::max(16, (M + 15) & ~15); }
bool stream_eligible(int M, int N, int epilogue) {
    if (!g_stream_enabled || M < 1 || M > 256) return false;
    return epilogue == kSwiGLU ? (N / 2) % kWRows == 0 : N % kWRows == 0;
}
int stream_nmma(int N, int epilogue) {
    if (epilogue == kSwiGLU) return 2;
    return (g_stream_nmma == 2 && N % (2 * kWRows) == 0) ? 2 : 1;
}
int64_t stream_slot_bytes(int M, int nmma) { return static_cast<int64_t>(nmma) * kWRows * stream_np(M) * 4; }

template <int EPI, int NMMA>
int launch_stream(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int64_t b_rows,
                  int n_tiles, int half_rows, uint16_t* c, int ldc, const uint16_t* r, void* ws, int64_t ws_bytes,
                  cudaStream_t stream) {
    StreamArgs p{};
    p.M = M;
    p.NP = stream_np(M);
    p.acc_stride = pow2ceil(std::max(32, p.NP));
    p.tmem_cols = static_cast<uint32_t>(std::max(32, NMMA * p.acc_stride));
    p.KB = K / BK;
    p.units = n_tiles * p.KB;
    const int stage_bytes = NMMA * kWTileBytes + p.NP * BK * 2;
    p.stages = std::min(8, kStreamSmemBudget / stage_bytes);
    if (p.stages < 2 || p.tmem_cols > 512) return KL_EUNSUPPORTED;
    int G = std::min(sm_count(), std::max(1, p.units / 4));
    G = static_cast<int>(std::min<int64_t>(G, (ws_bytes - kFlagBytes) / stream_slot_bytes(M, NMMA)));
    G = std::min(G, static_cast<int>(kFlagBytes / 4));
    if (G < 1) return KL_EUNSUPPORTED;
    p.half_rows = half_rows;
    p.c = c;
    p.ldc = ldc;
    p.r = r;
    p.flags = static_cast<uint32_t*>(ws);
    p.ws = reinterpret_cast<float*>(static_cast<char*>(ws) + kFlagBytes);
    p.epoch = next_epoch();
    CUtensorMap mw, mx;
    int rc = make_map(&mw, b, b_rows, K, kWRows);
    if (rc) return rc;
    rc = make_map(&mx, a, a_rows, K, p.NP);
    if (rc) return rc;
    const int smem = p.stages * stage_bytes + 1024 + 256;
    static bool configured = false;  // per template instance
    if (!configured) {
        KL_CUDA_TRY(cudaFuncSetAttribute(gemm_stream_kernel<EPI, NMMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kStreamSmemBudget + 1024 + 256));
        configured = true;
    }
    gemm_stream_kernel<EPI, NMMA><<<G, kStreamThreads, smem, stream>>>(mw, mx, static_cast<int>(row_offset), p);
    return check_launch();
}

int gemm_stream(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint16_t* b, int N,
                uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* ws, int64_t ws_bytes, cudaStream_t stream) {
    const int nmma = stream_nmma(N, epilogue);
    if (epilogue == kSwiGLU)
        return launch_stream<kSwiGLU, 2>(a, a_rows, row_offset, M, K, b, N, N / 2 / kWRows, N / 2, c, ldc, r, ws,
                                         ws_bytes, stream);
    const int n_tiles = N / (kWRows * nmma);
    if (epilogue == kResidual)
        return nmma == 2 ? launch_stream<kResidual, 2>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws,
                                                       ws_bytes, stream)
                         : launch_stream<kResidual, 1>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws,
                                                       ws_bytes, stream);
    return nmma == 2 ? launch_stream<kStore, 2>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws, ws_bytes,
                                                stream)
                     : launch_stream<kStore, 1>(a, a_rows, row_offset, M, K, b, N, n_tiles, 0, c, ldc, r, ws, ws_bytes,
                                                stream);
}

}  // namespace
}  // namespace kl

extern "C" int kl_tune(int knob, int value) {
    using namespace kl;
    switch (knob) {
        case KL_TUNE_STREAM_GEMM: g_stream_enabled = value != 0; return KL_OK;
        case KL_TUNE_STREAM_NMMA:
            if (value != 1 && value != 2) return KL_EINVAL;
            g_stream_nmma = value;
            return KL_OK;
        default: return KL_EINVAL;
    }
}

extern "C" int64_t kl_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
    using namespace kl;
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    if (stream_eligible(M, N, epilogue))
        return kFlagBytes + static_cast<int64_t>(sm_count()) * stream_slot_bytes(M, stream_nmma(N, epilogue));
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
    if (workspace != nullptr && stream_eligible(M, N, epilogue) &&
        workspace_bytes >= kFlagBytes + stream_slot_bytes(M, stream_nmma(N, epilogue))) {
        const int rc = gemm_stream(a, a_rows, row_offset, M, K, b, N, c, ldc, r, epilogue, workspace, workspace_bytes,
                                   stream);
        if (rc != KL_EUNSUPPORTED) return rc;
    }
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
