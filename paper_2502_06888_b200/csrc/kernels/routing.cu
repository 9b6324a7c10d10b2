// SPDX-License-Identifier: Apache-2.0
// Routing-path kernels (all HBM/latency bound, CUDA cores):
//   K1 kl_gate_topk      fused RMSNorm + router logits + top-k + weights +
//                        per-batch histogram / first-demand positions
//                        (reference op compute_gate, schedule.cpp:340-353;
//                         first-demand order = batch_demand, schedule.cpp:448-454)
//   K4 kl_permute        stable counting sort into expert-major rows
//                        (histogram = expert_load, trace.cpp:380-389)
//   K7 kl_combine        weighted sum of expert rows + residual
//   K2 kl_coact_update   co-activation counts (update_table, correlation.cpp:123-140)
//   K3 kl_predict_scores hist . C_j (predict_hot 'sum' scores, correlation.cpp:74-121)
//   kl_rmsnorm, kl_fill_normal_bf16
#include <cstdint>

#include "common.cuh"

namespace kl {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ void load8(const uint16_t* p, float (&v)[8]) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = bf2f(static_cast<uint16_t>(w[i] & 0xffffu));
        v[2 * i + 1] = bf2f(static_cast<uint16_t>(w[i] >> 16));
    }
}

// Warp-wide RMS of a bf16 row: sum of squares in a fixed order (lane-strided
// 8-element chunks, then xor butterfly), returns rsqrt(mean + eps).
__device__ __forceinline__ float row_rstd(const uint16_t* x, int d, float eps, int lane) {
    float ss = 0.f;
#pragma unroll 4
    for (int c = lane * 8; c < d; c += 256) {
        float v[8];
        load8(x + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    return rsqrtf(ss / static_cast<float>(d) + eps);
}

// Normalised row written as bf16: out = bf16((x * rstd) * w).
__device__ __forceinline__ void write_normed(const uint16_t* x, const uint16_t* w, uint16_t* out, int d, float rstd,
                                             int lane) {
#pragma unroll 4
    for (int c = lane * 8; c < d; c += 256) {
        float v[8], g[8];
        load8(x + c, v);
        load8(w + c, g);
        uint4 o;
        o.x = pack2(__fmul_rn(__fmul_rn(v[0], rstd), g[0]), __fmul_rn(__fmul_rn(v[1], rstd), g[1]));
        o.y = pack2(__fmul_rn(__fmul_rn(v[2], rstd), g[2]), __fmul_rn(__fmul_rn(v[3], rstd), g[3]));
        o.z = pack2(__fmul_rn(__fmul_rn(v[4], rstd), g[4]), __fmul_rn(__fmul_rn(v[5], rstd), g[5]));
        o.w = pack2(__fmul_rn(__fmul_rn(v[6], rstd), g[6]), __fmul_rn(__fmul_rn(v[7], rstd), g[7]));
        *reinterpret_cast<uint4*>(out + c) = o;
    }
}

// One CTA (kGateWarps warps) per token; warp w owns experts w, w+W, ...
// Logit order (mirrored in oracle/numerics.c): lane l accumulates fmaf over
// its chunks c = l*8 + 256*j, elements in order, then an xor butterfly
// 16,8,4,2,1 with round-to-nearest adds. Every warp recomputes the (bit-
// identical) normalised row in registers; warp 0 stores it as x2.
constexpr int kGateWarps = 4;

__global__ void __launch_bounds__(kGateWarps * 32)
gate_topk_kernel(const uint16_t* __restrict__ h, const uint16_t* __restrict__ norm_w,
                 const uint16_t* __restrict__ wg, int T, int d, int E, int k, float eps, int score_mode,
                 uint16_t* __restrict__ x2, float* __restrict__ logits_out, int32_t* __restrict__ idx,
                 float* __restrict__ weight, int32_t* __restrict__ hist, int32_t* __restrict__ first_pos) {
    pdl_enter();
    const int tok = blockIdx.x;
    const int wid = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint16_t* hrow = h + static_cast<int64_t>(tok) * d;
    const float rstd = row_rstd(hrow, d, eps, lane);
    if (wid == 0) write_normed(hrow, norm_w, x2 + static_cast<int64_t>(tok) * d, d, rstd, lane);

    __shared__ float lg[64];
    for (int e = wid; e < E; e += kGateWarps) {
        float acc = 0.f;
    #pragma unroll 4
    for (int c = lane * 8; c < d; c += 256) {
            float v[8], g[8], wv[8];
            load8(hrow + c, v);
            load8(norm_w + c, g);
            load8(wg + static_cast<int64_t>(e) * d + c, wv);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float xv = bf2f(f2bf(__fmul_rn(__fmul_rn(v[i], rstd), g[i])));
                acc = fmaf(xv, wv[i], acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if (lane == 0) lg[e] = acc;
    }
    __syncthreads();
    const int warp = tok;
    if (threadIdx.x != 0) return;
    if (logits_out != nullptr)
        for (int e = 0; e < E; ++e) logits_out[static_cast<int64_t>(warp) * E + e] = lg[e];
    // Top-k: repeated arg-max, strict '>' so ties keep the lower expert id.
    uint64_t taken = 0;
    int sel[8];
    float val[8];
    for (int j = 0; j < k; ++j) {
        int best = -1;
        float bv = 0.f;
        for (int e = 0; e < E; ++e) {
            if ((taken >> e) & 1ull) continue;
            if (best < 0 || lg[e] > bv) {
                best = e;
                bv = lg[e];
            }
        }
        taken |= 1ull << best;
        sel[j] = best;
        val[j] = bv;
    }
    float wsum = 0.f;
    float p[8];
    if (score_mode == 0) {
        for (int j = 0; j < k; ++j) {
            p[j] = expf(val[j] - val[0]);
            wsum += p[j];
        }
    } else {
        float mx = lg[0];
        for (int e = 1; e < E; ++e) mx = fmaxf(mx, lg[e]);
        for (int e = 0; e < E; ++e) wsum += expf(lg[e] - mx);
        for (int j = 0; j < k; ++j) p[j] = expf(val[j] - mx);
    }
    for (int j = 0; j < k; ++j) {
        const int64_t r = static_cast<int64_t>(warp) * k + j;
        idx[r] = sel[j];
        weight[r] = p[j] / wsum;
        if (hist != nullptr) atomicAdd(&hist[sel[j]], 1);
        if (first_pos != nullptr) atomicMin(&first_pos[sel[j]], static_cast<int32_t>(r));
    }
}

// Decode-sized router (few tokens): one 256-thread block per token so the
// token's E router rows are read by 8 warps at once. Every warp computes the
// row's RMSNorm itself, in the same order as gate_topk_warp_kernel (so x2
// and the logits are bit-identical to it and to the oracle), writes its
// eighth of x2, and dot-products the experts e = warp, warp + 8, ...; thread
// 0 then runs the same top-k / weights code.
template <int NC>
__global__ void __launch_bounds__(256)
gate_topk_block_kernel(uint16_t* h, const uint16_t* __restrict__ norm_w,
                       const uint16_t* __restrict__ wg, int T, int E, int k, float eps, int score_mode,
                       uint16_t* __restrict__ x2, float* __restrict__ logits_out, int32_t* __restrict__ idx,
                       float* __restrict__ weight, int32_t* __restrict__ hist, int32_t* __restrict__ first_pos,
                       const float* __restrict__ hpart, int S, int64_t part_split_elems,
                       unsigned long long* t_start, EndMark end) {
    pdl_enter();
    write_start_mark(t_start);
    constexpr int d = NC * 256;
    __shared__ float lg[64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tok = blockIdx.x;
    const uint16_t* hrow = h + static_cast<int64_t>(tok) * d;
    uint4 hv[NC];
    if (hpart != nullptr) {
        // Deferred o-proj: the row is first completed from the projection's
        // fp32 split partials (the owner's order: its own split S-1, then
        // 0..S-2) plus the residual, rounded once -- what the streaming
        // GEMM's residual epilogue would have stored -- and written back.
        __shared__ uint4 hrow_s[NC * 32];
        auto finish = [&](int j, int64_t off, float4 v0, float4 v1, uint4 r) {
            const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                o[e] = pack2(__fadd_rn(f[2 * e], bf2f(static_cast<uint16_t>(rw[e] & 0xffffu))),
                             __fadd_rn(f[2 * e + 1], bf2f(static_cast<uint16_t>(rw[e] >> 16))));
            const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
            hrow_s[j * 32 + lane] = ov;
            *reinterpret_cast<uint4*>(h + off) = ov;
        };
        auto add4 = [](float4& v, const float4& a) {
            v.x = __fadd_rn(v.x, a.x); v.y = __fadd_rn(v.y, a.y); v.z = __fadd_rn(v.z, a.z); v.w = __fadd_rn(v.w, a.w);
        };
        if (S <= 4) {
            // Every load of this warp's chunks issued before the first add
            // (slot 0 = the owner's split S-1, slot i = split i-1): one
            // memory latency instead of a chain of S x chunks.
            constexpr int kJ = (NC + 7) / 8;
            float4 pa[kJ][4][2];
            uint4 rr[kJ];
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int j = wid + 8 * jj;
                if (j >= NC) continue;
                const int64_t off = static_cast<int64_t>(tok) * d + lane * 8 + 256 * j;
#pragma unroll
                for (int sl = 0; sl < 4; ++sl)
                    if (sl < S) {
                        const int sp = sl == 0 ? S - 1 : sl - 1;
                        const float4* q = reinterpret_cast<const float4*>(hpart + sp * part_split_elems + off);
                        pa[jj][sl][0] = q[0];
                        pa[jj][sl][1] = q[1];
                    }
                rr[jj] = *reinterpret_cast<const uint4*>(h + off);
            }
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) {
                const int j = wid + 8 * jj;
                if (j >= NC) continue;
                float4 v0 = pa[jj][0][0], v1 = pa[jj][0][1];
#pragma unroll
                for (int sl = 1; sl < 4; ++sl)
                    if (sl < S) {
                        add4(v0, pa[jj][sl][0]);
                        add4(v1, pa[jj][sl][1]);
                    }
                finish(j, static_cast<int64_t>(tok) * d + lane * 8 + 256 * j, v0, v1, rr[jj]);
            }
        } else {
            for (int j = wid; j < NC; j += 8) {
                const int64_t off = static_cast<int64_t>(tok) * d + lane * 8 + 256 * j;
                const float4* own = reinterpret_cast<const float4*>(hpart + static_cast<int64_t>(S - 1) * part_split_elems + off);
                float4 v0 = own[0], v1 = own[1];
                for (int sp = 0; sp < S - 1; ++sp) {
                    const float4* q = reinterpret_cast<const float4*>(hpart + sp * part_split_elems + off);
                    add4(v0, q[0]);
                    add4(v1, q[1]);
                }
                finish(j, off, v0, v1, *reinterpret_cast<const uint4*>(h + off));
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NC; ++j) hv[j] = hrow_s[j * 32 + lane];
    } else {
#pragma unroll
        for (int j = 0; j < NC; ++j) hv[j] = __ldg(reinterpret_cast<const uint4*>(hrow + lane * 8 + 256 * j));
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const uint32_t w4[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = bf2f(static_cast<uint16_t>(w4[i] & 0xffffu)), b = bf2f(static_cast<uint16_t>(w4[i] >> 16));
            ss = fmaf(a, a, ss);
            ss = fmaf(b, b, ss);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    const float rstd = rsqrtf(ss / static_cast<float>(d) + eps);
    uint32_t xv[NC][4];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(norm_w + lane * 8 + 256 * j));
        const uint32_t hw[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
        const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = __fmul_rn(__fmul_rn(bf2f(static_cast<uint16_t>(hw[i] & 0xffffu)), rstd),
                                      bf2f(static_cast<uint16_t>(gw[i] & 0xffffu)));
            const float b = __fmul_rn(__fmul_rn(bf2f(static_cast<uint16_t>(hw[i] >> 16)), rstd),
                                      bf2f(static_cast<uint16_t>(gw[i] >> 16)));
            xv[j][i] = pack2(a, b);
        }
        if ((j & 7) == wid)
            *reinterpret_cast<uint4*>(x2 + static_cast<int64_t>(tok) * d + lane * 8 + 256 * j) =
                make_uint4(xv[j][0], xv[j][1], xv[j][2], xv[j][3]);
    }
    for (int e = wid; e < E; e += 8) {
        const uint16_t* wr = wg + static_cast<int64_t>(e) * d + lane * 8;
        uint4 wv[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) wv[j] = __ldg(reinterpret_cast<const uint4*>(wr + 256 * j));
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const uint32_t ww[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc = fmaf(bf2f(static_cast<uint16_t>(xv[j][i] & 0xffffu)), bf2f(static_cast<uint16_t>(ww[i] & 0xffffu)), acc);
                acc = fmaf(bf2f(static_cast<uint16_t>(xv[j][i] >> 16)), bf2f(static_cast<uint16_t>(ww[i] >> 16)), acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if (lane == 0) lg[e] = acc;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (logits_out != nullptr)
        for (int e = 0; e < E; ++e) logits_out[static_cast<int64_t>(tok) * E + e] = lg[e];
    uint64_t taken = 0;
    int sel[8];
    float val[8];
    for (int j = 0; j < k; ++j) {
        int best = -1;
        float bv = 0.f;
        for (int e = 0; e < E; ++e) {
            if ((taken >> e) & 1ull) continue;
            if (best < 0 || lg[e] > bv) {
                best = e;
                bv = lg[e];
            }
        }
        taken |= 1ull << best;
        sel[j] = best;
        val[j] = bv;
    }
    float wsum = 0.f;
    float pr[8];
    if (score_mode == 0) {
        for (int j = 0; j < k; ++j) {
            pr[j] = expf(val[j] - val[0]);
            wsum += pr[j];
        }
    } else {
        float mx = lg[0];
        for (int e = 1; e < E; ++e) mx = fmaxf(mx, lg[e]);
        for (int e = 0; e < E; ++e) wsum += expf(lg[e] - mx);
        for (int j = 0; j < k; ++j) pr[j] = expf(val[j] - mx);
    }
    for (int j = 0; j < k; ++j) {
        const int64_t r = static_cast<int64_t>(tok) * k + j;
        idx[r] = sel[j];
        weight[r] = pr[j] / wsum;
        if (hist != nullptr) atomicAdd(&hist[sel[j]], 1);
        if (first_pos != nullptr) atomicMin(&first_pos[sel[j]], static_cast<int32_t>(r));
    }
    write_end_mark(end.t, end.cnt);  // thread 0: the block's last live thread
}

// Latency-optimised router: one warp per token, the row held in registers
// (NC = d/256 16-byte chunks per lane, loaded once), every expert's router row
// loaded with independent vector loads. Same arithmetic order as
// gate_topk_kernel (and oracle/numerics.c): lane l owns chunks c = 8l + 256j,
// fmaf in element order, xor butterfly 16..1 with round-to-nearest adds.
template <int NC>
__global__ void __launch_bounds__(128)
gate_topk_warp_kernel(const uint16_t* __restrict__ h, const uint16_t* __restrict__ norm_w,
                      const uint16_t* __restrict__ wg, int T, int E, int k, float eps, int score_mode,
                      uint16_t* __restrict__ x2, float* __restrict__ logits_out, int32_t* __restrict__ idx,
                      float* __restrict__ weight, int32_t* __restrict__ hist, int32_t* __restrict__ first_pos) {
    pdl_enter();
    constexpr int d = NC * 256;
    __shared__ float lg_all[4][64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tok = blockIdx.x * 4 + wid;
    if (tok >= T) return;
    const uint16_t* hrow = h + static_cast<int64_t>(tok) * d;
    uint4 hv[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) hv[j] = __ldg(reinterpret_cast<const uint4*>(hrow + lane * 8 + 256 * j));
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const uint32_t w4[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = bf2f(static_cast<uint16_t>(w4[i] & 0xffffu)), b = bf2f(static_cast<uint16_t>(w4[i] >> 16));
            ss = fmaf(a, a, ss);
            ss = fmaf(b, b, ss);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    const float rstd = rsqrtf(ss / static_cast<float>(d) + eps);
    // Normalised row (bf16, as stored in x2) kept packed in registers.
    uint32_t xv[NC][4];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(norm_w + lane * 8 + 256 * j));
        const uint32_t hw[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
        const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = __fmul_rn(__fmul_rn(bf2f(static_cast<uint16_t>(hw[i] & 0xffffu)), rstd),
                                      bf2f(static_cast<uint16_t>(gw[i] & 0xffffu)));
            const float b = __fmul_rn(__fmul_rn(bf2f(static_cast<uint16_t>(hw[i] >> 16)), rstd),
                                      bf2f(static_cast<uint16_t>(gw[i] >> 16)));
            xv[j][i] = pack2(a, b);
        }
        *reinterpret_cast<uint4*>(x2 + static_cast<int64_t>(tok) * d + lane * 8 + 256 * j) =
            make_uint4(xv[j][0], xv[j][1], xv[j][2], xv[j][3]);
    }
    float* lg = lg_all[wid];
    for (int e = 0; e < E; ++e) {
        const uint16_t* wr = wg + static_cast<int64_t>(e) * d + lane * 8;
        uint4 wv[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) wv[j] = __ldg(reinterpret_cast<const uint4*>(wr + 256 * j));
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const uint32_t ww[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc = fmaf(bf2f(static_cast<uint16_t>(xv[j][i] & 0xffffu)), bf2f(static_cast<uint16_t>(ww[i] & 0xffffu)), acc);
                acc = fmaf(bf2f(static_cast<uint16_t>(xv[j][i] >> 16)), bf2f(static_cast<uint16_t>(ww[i] >> 16)), acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        if (lane == 0) lg[e] = acc;
    }
    __syncwarp();
    if (lane != 0) return;
    if (logits_out != nullptr)
        for (int e = 0; e < E; ++e) logits_out[static_cast<int64_t>(tok) * E + e] = lg[e];
    uint64_t taken = 0;
    int sel[8];
    float val[8];
    for (int j = 0; j < k; ++j) {
        int best = -1;
        float bv = 0.f;
        for (int e = 0; e < E; ++e) {
            if ((taken >> e) & 1ull) continue;
            if (best < 0 || lg[e] > bv) {
                best = e;
                bv = lg[e];
            }
        }
        taken |= 1ull << best;
        sel[j] = best;
        val[j] = bv;
    }
    float wsum = 0.f;
    float pr[8];
    if (score_mode == 0) {
        for (int j = 0; j < k; ++j) {
            pr[j] = expf(val[j] - val[0]);
            wsum += pr[j];
        }
    } else {
        float mx = lg[0];
        for (int e = 1; e < E; ++e) mx = fmaxf(mx, lg[e]);
        for (int e = 0; e < E; ++e) wsum += expf(lg[e] - mx);
        for (int j = 0; j < k; ++j) pr[j] = expf(val[j] - mx);
    }
    for (int j = 0; j < k; ++j) {
        const int64_t r = static_cast<int64_t>(tok) * k + j;
        idx[r] = sel[j];
        weight[r] = pr[j] / wsum;
        if (hist != nullptr) atomicAdd(&hist[sel[j]], 1);
        if (first_pos != nullptr) atomicMin(&first_pos[sel[j]], static_cast<int32_t>(r));
    }
}

__global__ void rmsnorm_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int64_t T, int d,
                               float eps, uint16_t* __restrict__ out) {
    pdl_enter();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= T) return;
    const float rstd = row_rstd(x + row * d, d, eps, lane);
    write_normed(x + row * d, w, out + row * d, d, rstd, lane);
}

// Few rows (decode): one 8-warp block per row; every warp computes the
// row's rstd (same order, bit-identical) and writes every 8th 256-column
// span, so a 64-row call spreads over 64 SMs instead of 16.
__global__ void __launch_bounds__(256)
rmsnorm_row_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int d, float eps,
                   uint16_t* __restrict__ out, const int32_t* __restrict__ rope_pos, float rope_theta, int rope_hd,
                   float2* __restrict__ rope_table, unsigned long long* t_start) {
    pdl_enter();
    write_start_mark(t_start);
    if (rope_table != nullptr && static_cast<int>(threadIdx.x) < rope_hd / 2) {
        // This token's RoPE cos/sin table for the QKV GEMM's fused epilogue.
        float cs, sn;
        rope_cs(rope_pos[blockIdx.x], threadIdx.x, rope_hd, rope_theta, cs, sn);
        rope_table[static_cast<int64_t>(blockIdx.x) * (rope_hd / 2) + threadIdx.x] = make_float2(cs, sn);
    }
    // (pdl_enter released the QKV GEMM that follows: it may start now and
    // prefetch its weights; it reads this kernel's output only after
    // griddepcontrol.wait.)
    const int64_t row = blockIdx.x;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float rstd = row_rstd(x + row * d, d, eps, lane);
    const uint16_t* xr = x + row * d;
    uint16_t* orow = out + row * d;
    for (int c = wid * 256 + lane * 8; c < d; c += 8 * 256) {
        float v[8], g[8];
        load8(xr + c, v);
        load8(w + c, g);
        uint4 o;
        o.x = pack2(__fmul_rn(__fmul_rn(v[0], rstd), g[0]), __fmul_rn(__fmul_rn(v[1], rstd), g[1]));
        o.y = pack2(__fmul_rn(__fmul_rn(v[2], rstd), g[2]), __fmul_rn(__fmul_rn(v[3], rstd), g[3]));
        o.z = pack2(__fmul_rn(__fmul_rn(v[4], rstd), g[4]), __fmul_rn(__fmul_rn(v[5], rstd), g[5]));
        o.w = pack2(__fmul_rn(__fmul_rn(v[6], rstd), g[6]), __fmul_rn(__fmul_rn(v[7], rstd), g[7]));
        *reinterpret_cast<uint4*>(orow + c) = o;
    }
}

// ---------------------------------------------------------------- permute --
// Chunk of 1024 routed rows per CTA (32 warps): per-warp match_any ranks,
// per-expert warp prefix in smem -> stable local rank within the chunk.
constexpr int kChunk = 1024;

__global__ void __launch_bounds__(kChunk)
permute_rank_kernel(const int32_t* __restrict__ idx, int64_t R, int E, int32_t* __restrict__ chunk_counts,
                    int32_t* __restrict__ local_rank, int32_t* __restrict__ counts, int32_t* __restrict__ offsets) {
    pdl_enter();
    __shared__ int32_t warp_cnt[32][64];
    __shared__ int32_t tot[64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kChunk + threadIdx.x;
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) (&warp_cnt[0][0])[i] = 0;
    __syncthreads();
    const bool valid = r < R;
    const int e = valid ? idx[r] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) warp_cnt[warp][e] = __popc(peers);
    __syncthreads();
    // Exclusive prefix over warps per expert (thread e scans column e).
    if (threadIdx.x < E) {
        int run = 0;
        for (int w = 0; w < 32; ++w) {
            const int c = warp_cnt[w][threadIdx.x];
            warp_cnt[w][threadIdx.x] = run;
            run += c;
        }
        chunk_counts[static_cast<int64_t>(blockIdx.x) * E + threadIdx.x] = run;
        tot[threadIdx.x] = run;
    }
    __syncthreads();
    if (valid) local_rank[r] = warp_cnt[warp][e] + rank;
    if (offsets != nullptr && threadIdx.x < 32) {
        // Single chunk (decode-sized calls): the scan kernel's work in the
        // same launch. Chunk base of expert e = its exclusive offset.
        int run = 0;
        for (int base = 0; base < E; base += 32) {
            const int e2 = base + threadIdx.x;
            const int v = e2 < E ? tot[e2] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (threadIdx.x >= o) incl += y;
            }
            if (e2 < E) {
                const int excl = run + incl - v;
                offsets[e2] = excl;
                chunk_counts[e2] = excl;
                if (counts != nullptr) counts[e2] = v;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (threadIdx.x == 0) offsets[E] = run;
    }
}

// One thread per expert: totals, exclusive offsets, per-chunk bases.
__global__ void permute_scan_kernel(int32_t* __restrict__ chunk_counts, int64_t n_chunks, int E,
                                    int32_t* __restrict__ counts, int32_t* __restrict__ offsets) {
    pdl_enter();
    __shared__ int32_t total[64];
    const int e = threadIdx.x;
    if (e < E) {
        int32_t run = 0;
        for (int64_t c = 0; c < n_chunks; ++c) {
            const int32_t v = chunk_counts[c * E + e];
            chunk_counts[c * E + e] = run;  // becomes the within-expert chunk base
            run += v;
        }
        total[e] = run;
        if (counts != nullptr) counts[e] = run;
    }
    __syncthreads();
    if (e == 0) {
        int32_t acc = 0;
        for (int i = 0; i < E; ++i) {
            offsets[i] = acc;
            acc += total[i];
        }
        offsets[E] = acc;
    }
    __syncthreads();
    if (e < E) {
        const int32_t base = offsets[e];
        for (int64_t c = 0; c < n_chunks; ++c) chunk_counts[c * E + e] += base;
    }
}

// One CTA of kRowThreads per routed row: position and inverse map (thread
// 0), then the 16-byte row copy with every load of a group issued before its
// stores (a row is d*2 bytes: 8 KB at d = 4096, 4 x 16 B per thread), so a
// decode-sized call keeps the whole copy in flight at once instead of one
// warp-serial 16 B chain per row.
constexpr int kRowThreads = 128;
constexpr int kRowGroup = 4;  // 16-byte chunks per thread in flight

__global__ void __launch_bounds__(kRowThreads)
permute_scatter_kernel(const int32_t* __restrict__ idx, int64_t R, int k, int E,
                       const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ local_rank,
                       const uint16_t* __restrict__ x2, int d, int32_t* __restrict__ pos,
                       int32_t* __restrict__ row_token, uint16_t* __restrict__ xp) {
    pdl_enter();
    const int64_t r = blockIdx.x;
    if (r >= R) return;
    const int e = idx[r];
    const int32_t p = chunk_base[(r / kChunk) * E + e] + local_rank[r];
    const int64_t t = r / k;
    if (threadIdx.x == 0) {
        pos[r] = p;
        if (row_token != nullptr) row_token[p] = static_cast<int32_t>(t);
    }
    if (xp == nullptr) return;
    const uint4* src = reinterpret_cast<const uint4*>(x2 + t * d);
    uint4* dst = reinterpret_cast<uint4*>(xp + static_cast<int64_t>(p) * d);
    const int n16 = d / 8;
    for (int g = 0; g < n16; g += kRowThreads * kRowGroup) {
        uint4 v[kRowGroup];
#pragma unroll
        for (int u = 0; u < kRowGroup; ++u) {
            const int i = g + u * kRowThreads + threadIdx.x;
            if (i < n16) v[u] = __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < kRowGroup; ++u) {
            const int i = g + u * kRowThreads + threadIdx.x;
            if (i < n16) dst[i] = v[u];
        }
    }
}

// ---------------------------------------------------------------- combine --
// out[t] = resid[t] + sum_j w[t,j] * y[pos[t,j]]  (fp32 fma in j order, one
// rounding), one CTA of kRowThreads per token. Each thread owns up to
// kRowGroup 8-column chunks of the row per pass and issues all of their
// loads (residual + k gathered expert rows) before any arithmetic or store;
// out may alias resid (the engine combines in place), which is safe because
// a thread only stores the chunks it has already loaded.
template <int KMAX>
__global__ void __launch_bounds__(kRowThreads)
combine_kernel(const uint16_t* __restrict__ y, const int32_t* __restrict__ pos, const float* __restrict__ weight,
               const uint16_t* resid, int64_t T, int k, int d, uint16_t* out) {
    pdl_enter();
    const int64_t t = blockIdx.x;
    if (t >= T) return;
    int32_t p[KMAX];
    float w[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        p[j] = j < k ? pos[t * k + j] : 0;
        w[j] = j < k ? weight[t * k + j] : 0.f;
    }
    const int n8 = d / 8;
    for (int g = 0; g < n8; g += kRowThreads * kRowGroup) {
        uint4 rq[kRowGroup];
        uint4 yq[kRowGroup][KMAX];
#pragma unroll
        for (int u = 0; u < kRowGroup; ++u) {
            const int i = g + u * kRowThreads + threadIdx.x;
            if (i < n8) {
                rq[u] = *reinterpret_cast<const uint4*>(resid + t * d + i * 8);
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                    if (j < k) yq[u][j] = __ldg(reinterpret_cast<const uint4*>(y + static_cast<int64_t>(p[j]) * d) + i);
            }
        }
#pragma unroll
        for (int u = 0; u < kRowGroup; ++u) {
            const int i = g + u * kRowThreads + threadIdx.x;
            if (i >= n8) continue;
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < KMAX; ++j) {
                if (j >= k) break;
                const uint32_t yw[4] = {yq[u][j].x, yq[u][j].y, yq[u][j].z, yq[u][j].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] = fmaf(w[j], bf2f(static_cast<uint16_t>(yw[q] & 0xffffu)), acc[2 * q]);
                    acc[2 * q + 1] = fmaf(w[j], bf2f(static_cast<uint16_t>(yw[q] >> 16)), acc[2 * q + 1]);
                }
            }
            const uint32_t rw[4] = {rq[u].x, rq[u].y, rq[u].z, rq[u].w};
            float rv[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                rv[2 * q] = bf2f(static_cast<uint16_t>(rw[q] & 0xffffu));
                rv[2 * q + 1] = bf2f(static_cast<uint16_t>(rw[q] >> 16));
            }
            uint4 o;
            o.x = pack2(__fadd_rn(rv[0], acc[0]), __fadd_rn(rv[1], acc[1]));
            o.y = pack2(__fadd_rn(rv[2], acc[2]), __fadd_rn(rv[3], acc[3]));
            o.z = pack2(__fadd_rn(rv[4], acc[4]), __fadd_rn(rv[5], acc[5]));
            o.w = pack2(__fadd_rn(rv[6], acc[6]), __fadd_rn(rv[7], acc[7]));
            *reinterpret_cast<uint4*>(out + t * d + i * 8) = o;
        }
    }
}

// combine_kernel over a down projection left as S fp32 split partials
// (kl_expert_ffn_kb_deferred): y = bf16(((p[S-1] + p[0]) + p[1]) + ...), the
// order the streaming GEMM's owner would have summed them in (its own split
// last in the k range, then the contributors ascending), then the same
// weighted sum as combine_kernel: bit-identical to the non-deferred path.
template <int KMAX>
__global__ void __launch_bounds__(kRowThreads)
combine_deferred_kernel(const float* __restrict__ yp, int S, int64_t split_elems, const int32_t* __restrict__ pos,
                        const float* __restrict__ weight, const uint16_t* resid, int64_t T, int k, int d,
                        uint16_t* out) {
    pdl_enter();
    const int64_t t = blockIdx.x;
    if (t >= T) return;
    int32_t p[KMAX];
    float w[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        p[j] = j < k ? pos[t * k + j] : 0;
        w[j] = j < k ? weight[t * k + j] : 0.f;
    }
    const int n8 = d / 8;
    for (int i = threadIdx.x; i < n8; i += kRowThreads) {
        const uint4 rq = *reinterpret_cast<const uint4*>(resid + t * d + i * 8);
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        // Up to two routed rows' partials loaded before the first add (one
        // memory latency per pair of rows instead of one per row).
#pragma unroll
        for (int j0 = 0; j0 < KMAX; j0 += 2) {
            if (j0 >= k) break;
            float4 o0[2], o1[2], q0[2][3], q1[2][3];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = j0 + jj;
                if (j >= k) break;
                const float* base = yp + static_cast<int64_t>(p[j]) * d + i * 8;
                const float4* own = reinterpret_cast<const float4*>(base + static_cast<int64_t>(S - 1) * split_elems);
                o0[jj] = __ldg(own);
                o1[jj] = __ldg(own + 1);
#pragma unroll
                for (int sp = 0; sp < 3; ++sp)
                    if (sp < S - 1) {
                        const float4* src = reinterpret_cast<const float4*>(base + sp * split_elems);
                        q0[jj][sp] = __ldg(src);
                        q1[jj][sp] = __ldg(src + 1);
                    }
            }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = j0 + jj;
                if (j >= k) break;
                float y[8] = {o0[jj].x, o0[jj].y, o0[jj].z, o0[jj].w, o1[jj].x, o1[jj].y, o1[jj].z, o1[jj].w};
#pragma unroll
                for (int sp = 0; sp < 3; ++sp) {
                    if (sp >= S - 1) break;
                    const float q[8] = {q0[jj][sp].x, q0[jj][sp].y, q0[jj][sp].z, q0[jj][sp].w,
                                        q1[jj][sp].x, q1[jj][sp].y, q1[jj][sp].z, q1[jj][sp].w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) y[e] = __fadd_rn(y[e], q[e]);
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] = fmaf(w[j], bf2f(f2bf(y[e])), acc[e]);
            }
        }
        const uint32_t rw[4] = {rq.x, rq.y, rq.z, rq.w};
        float rv[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            rv[2 * q] = bf2f(static_cast<uint16_t>(rw[q] & 0xffffu));
            rv[2 * q + 1] = bf2f(static_cast<uint16_t>(rw[q] >> 16));
        }
        uint4 o;
        o.x = pack2(__fadd_rn(rv[0], acc[0]), __fadd_rn(rv[1], acc[1]));
        o.y = pack2(__fadd_rn(rv[2], acc[2]), __fadd_rn(rv[3], acc[3]));
        o.z = pack2(__fadd_rn(rv[4], acc[4]), __fadd_rn(rv[5], acc[5]));
        o.w = pack2(__fadd_rn(rv[6], acc[6]), __fadd_rn(rv[7], acc[7]));
        *reinterpret_cast<uint4*>(out + t * d + i * 8) = o;
    }
}

// ------------------------------------------------------------ prefetcher --
__global__ void coact_kernel(const int32_t* __restrict__ prev, const int32_t* __restrict__ cur, int64_t T, int k,
                             int E, int layer, int64_t* __restrict__ table, int64_t* __restrict__ marginal) {
    pdl_enter();
    extern __shared__ int32_t cnt[];  // E*E (or E for the marginal)
    const int cells = layer == 0 ? E : E * E;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < T;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (layer == 0) {
            for (int j = 0; j < k; ++j) atomicAdd(&cnt[cur[t * k + j]], 1);
        } else {
            for (int a = 0; a < k; ++a) {
                const int pa = prev[t * k + a];
                for (int b = 0; b < k; ++b) atomicAdd(&cnt[pa * E + cur[t * k + b]], 1);
            }
        }
    }
    __syncthreads();
    int64_t* dst = layer == 0 ? marginal : table + static_cast<int64_t>(layer - 1) * E * E;
    for (int i = threadIdx.x; i < cells; i += blockDim.x)
        if (cnt[i] != 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(dst + i), static_cast<unsigned long long>(cnt[i]));
}

__global__ void predict_kernel(const int32_t* __restrict__ hist, const int64_t* __restrict__ table, int E,
                               int layer, int64_t* __restrict__ score) {
    pdl_enter();
    const int b = threadIdx.x;
    if (b >= E) return;
    const int64_t* tab = table + static_cast<int64_t>(layer - 1) * E * E;
    int64_t s = 0;
    for (int a = 0; a < E; ++a) s += static_cast<int64_t>(hist[a]) * tab[a * E + b];
    score[b] = s;
}

// ------------------------------------------------------------ synthetic init --
__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// Approximately normal values with bit-reproducible arithmetic: Irwin-Hall
// sum of four 22-bit uniforms (exact in fp32), centred and scaled by
// sqrt(3)*std (one correctly rounded multiply), so the CPU oracle
// regenerates identical bf16 weights from (seed, index).
__global__ void fill_normal_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t seed, float sd) {
    const float scale = 1.7320508075688772f * sd;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t z = splitmix(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ULL));
        const uint64_t w = splitmix(z);
        const float u = __fadd_rn(__fadd_rn(static_cast<float>(z & 0x3fffffu), static_cast<float>((z >> 22) & 0x3fffffu)),
                                  __fadd_rn(static_cast<float>(w & 0x3fffffu), static_cast<float>((w >> 22) & 0x3fffffu)));
        const float c = __fsub_rn(__fmul_rn(u, 0x1.0p-22f), 2.0f);
        dst[i] = f2bf(__fmul_rn(c, scale));
    }
}

// Replay routing: force the trace's ids, recompute weights from the router's
// own logits of those ids (mode-0 softmax) and the batch histograms.
__global__ void route_override_kernel(const int32_t* __restrict__ forced, const float* __restrict__ logits, int T,
                                      int E, int k, int32_t* __restrict__ idx, float* __restrict__ weight,
                                      int32_t* __restrict__ hist, int32_t* __restrict__ first_pos) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    float v[8], mx = -INFINITY, sum = 0.f;
    for (int j = 0; j < k; ++j) {
        const int e = forced[static_cast<int64_t>(t) * k + j];
        v[j] = logits[static_cast<int64_t>(t) * E + e];
        mx = j == 0 ? v[j] : mx;
    }
    for (int j = 0; j < k; ++j) sum += (v[j] = expf(v[j] - mx));
    for (int j = 0; j < k; ++j) {
        const int64_t r = static_cast<int64_t>(t) * k + j;
        const int e = forced[r];
        idx[r] = e;
        weight[r] = v[j] / sum;
        if (hist != nullptr) atomicAdd(&hist[e], 1);
        if (first_pos != nullptr) atomicMin(&first_pos[e], static_cast<int32_t>(r));
    }
}

__global__ void embed_kernel(const int32_t* __restrict__ ids, const uint16_t* __restrict__ table, int64_t T, int d,
                             uint16_t* __restrict__ out) {
    pdl_enter();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= T) return;
    const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<int64_t>(ids[t]) * d);
    uint4* dst = reinterpret_cast<uint4*>(out + t * d);
#pragma unroll 4
    for (int i = lane; i < d / 8; i += 32) dst[i] = __ldg(src + i);
}

// Greedy decode: first index of the row maximum (bf16 logits).
__global__ void argmax_kernel(const uint16_t* __restrict__ logits, int64_t T, int V, int32_t* __restrict__ out) {
    pdl_enter();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= T) return;
    const uint16_t* row = logits + t * V;
    float best = -INFINITY;
    int arg = 0x7fffffff;
    for (int i = lane; i < V; i += 32) {
        const float v = bf2f(row[i]);
        if (v > best) {
            best = v;
            arg = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    if (lane == 0) out[t] = arg;
}

int grid_for(int64_t items, int per_block) {
    const int64_t g = (items + per_block - 1) / per_block;
    return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace kl

using namespace kl;

extern "C" int kl_gate_topk(const uint16_t* h, const uint16_t* norm_w, const uint16_t* wg, int T, int d, int E, int k,
                            float eps, int score_mode, uint16_t* x2, float* logits, int32_t* idx, float* weight,
                            int32_t* hist, int32_t* first_pos, cudaStream_t stream) {
    if (T < 0 || d <= 0 || d % 256 != 0 || E < 1 || E > 64 || k < 1 || k > 8 || k > E) return KL_EINVAL;
    if (!h || !norm_w || !wg || !x2 || !idx || !weight) return KL_EINVAL;
    if (T == 0) return KL_OK;
    const unsigned blocks = static_cast<unsigned>((T + 3) / 4);
    // Few tokens (decode): a block per token fills more SMs and keeps 8 router
    // rows in flight per token; many tokens (prefill): a warp per token.
    const bool per_block = T <= 4 * 148;
#define KL_GATE_WARP(NC)                                                                                          \
    case NC:                                                                                                      \
        if (per_block)                                                                                            \
            return launch_pdl(gate_topk_block_kernel<NC>, dim3(static_cast<unsigned>(T)), dim3(256), 0, stream,   \
                              const_cast<uint16_t*>(h), norm_w, wg, T, E, k, eps, score_mode, x2, logits, idx,       \
                              weight, hist, first_pos, static_cast<const float*>(nullptr), 0, int64_t{0},            \
                              take_next_start(), take_next_end());                                                 \
        if (unsigned long long* ts = take_next_start())                                                           \
            if (const int rc = kl_stamp(ts, stream)) return rc;                                                   \
        return launch_pdl(gate_topk_warp_kernel<NC>, dim3(blocks), dim3(128), 0, stream, h, norm_w, wg, T, E, k, eps, \
                          score_mode, x2, logits, idx, weight, hist, first_pos);
    switch (d / 256) {
        KL_GATE_WARP(2)
        KL_GATE_WARP(4)
        KL_GATE_WARP(8)
        KL_GATE_WARP(16)
        KL_GATE_WARP(24)
        default: break;
    }
#undef KL_GATE_WARP
    if (unsigned long long* ts = take_next_start())
        if (const int rc = kl_stamp(ts, stream)) return rc;
    return launch_pdl(gate_topk_kernel, dim3(T), dim3(kGateWarps * 32), 0, stream, h, norm_w, wg, T, d, E, k, eps,
                      score_mode, x2, logits, idx, weight, hist, first_pos);
}

extern "C" int kl_gate_topk_deferred(uint16_t* h, const float* h_part, int splits, int64_t part_rows,
                                     const uint16_t* norm_w, const uint16_t* wg, int T, int d, int E, int k, float eps,
                                     int score_mode, uint16_t* x2, float* logits, int32_t* idx, float* weight,
                                     int32_t* hist, int32_t* first_pos, cudaStream_t stream) {
    if (T < 0 || d <= 0 || d % 256 != 0 || E < 1 || E > 64 || k < 1 || k > 8 || k > E) return KL_EINVAL;
    if (!h || !h_part || !norm_w || !wg || !x2 || !idx || !weight || splits < 1 || splits > 4 || T > part_rows)
        return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (T > 4 * 148) return KL_EUNSUPPORTED;  // decode-sized calls (block per token) only
    const int64_t pse = part_rows * d;
#define KL_GATE_DEF(NC)                                                                                           \
    case NC:                                                                                                      \
        return launch_pdl(gate_topk_block_kernel<NC>, dim3(static_cast<unsigned>(T)), dim3(256), 0, stream, h,     \
                          norm_w, wg, T, E, k, eps, score_mode, x2, logits, idx, weight, hist, first_pos, h_part,   \
                          splits, pse, take_next_start(), take_next_end());
    switch (d / 256) {
        KL_GATE_DEF(2)
        KL_GATE_DEF(4)
        KL_GATE_DEF(8)
        KL_GATE_DEF(16)
        KL_GATE_DEF(24)
        default: break;
    }
#undef KL_GATE_DEF
    return KL_EUNSUPPORTED;
}

extern "C" int kl_rmsnorm(const uint16_t* x, const uint16_t* w, int64_t T, int d, float eps, uint16_t* out,
                          cudaStream_t stream) {
    if (T < 0 || d <= 0 || d % 256 != 0 || !x || !w || !out) return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (T <= 4 * 148)
        return launch_pdl(rmsnorm_row_kernel, dim3(static_cast<unsigned>(T)), dim3(256), 0, stream, x, w, d, eps, out,
                          static_cast<const int32_t*>(nullptr), 0.0f, 0, static_cast<float2*>(nullptr),
                          take_next_start());
    if (unsigned long long* ts = take_next_start())
        if (const int rc = kl_stamp(ts, stream)) return rc;
    return launch_pdl(rmsnorm_kernel, dim3(grid_for(T, kWarpsPerBlock)), dim3(kWarpsPerBlock * 32), 0, stream, x, w, T,
                      d, eps, out);
}

extern "C" int kl_rmsnorm_rope_table(const uint16_t* x, const uint16_t* w, int64_t T, int d, float eps, uint16_t* out,
                                     const int32_t* pos, float theta, int hd, float* table, cudaStream_t stream) {
    if (T < 0 || d <= 0 || d % 256 != 0 || !x || !w || !out || !pos || !table || hd < 2 || hd > 512 || hd % 2)
        return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (T > 4 * 148) return KL_EUNSUPPORTED;  // decode-sized calls (block per row) only
    return launch_pdl(rmsnorm_row_kernel, dim3(static_cast<unsigned>(T)), dim3(256), 0, stream, x, w, d, eps, out, pos,
                      theta, hd, reinterpret_cast<float2*>(table), take_next_start());
}

extern "C" int64_t kl_permute_workspace_bytes(int64_t R, int E) {
    const int64_t chunks = (R + kChunk - 1) / kChunk;
    return (chunks * E + R) * static_cast<int64_t>(sizeof(int32_t)) + 256;
}

extern "C" int kl_permute_launches(int64_t R) { return R == 0 ? 1 : (R <= kChunk ? 2 : 3); }

extern "C" int kl_permute(const int32_t* idx, int64_t T, int k, int E, const uint16_t* x2, int d, int32_t* counts,
                          int32_t* offsets, int32_t* pos, int32_t* row_token, uint16_t* xp, void* workspace,
                          cudaStream_t stream) {
    if (T < 0 || k < 1 || E < 1 || E > 64 || !idx || !offsets || !pos || !workspace) return KL_EINVAL;
    if (xp != nullptr && (x2 == nullptr || d % 8 != 0)) return KL_EINVAL;
    const int64_t R = T * k;
    const int64_t chunks = (R + kChunk - 1) / kChunk;
    int32_t* chunk_counts = static_cast<int32_t*>(workspace);
    int32_t* local_rank = chunk_counts + chunks * E;
    if (R > 0) {
        // One chunk: rank + scan in a single launch.
        if (int rc_ = launch_pdl(permute_rank_kernel, dim3(static_cast<int>(chunks)), dim3(kChunk), 0, stream, idx, R, E, chunk_counts, local_rank, chunks == 1 ? counts : nullptr, chunks == 1 ? offsets : nullptr)) return rc_;
        KL_CUDA_TRY(cudaGetLastError());
    }
    if (chunks != 1) {
        if (int rc_ = launch_pdl(permute_scan_kernel, dim3(1), dim3(64), 0, stream, chunk_counts, chunks, E, counts, offsets)) return rc_;
        KL_CUDA_TRY(cudaGetLastError());
    }
    if (R == 0) return KL_OK;
    if (int rc_ = launch_pdl(permute_scatter_kernel, dim3(static_cast<unsigned>(R)), dim3(kRowThreads), 0, stream, idx, R, k, E, chunk_counts,
                                                                                local_rank, x2, d, pos, row_token, xp)) return rc_;
    return check_launch();
}

extern "C" int kl_combine(const uint16_t* y, const int32_t* pos, const float* weight, const uint16_t* resid, int64_t T,
                          int k, int d, uint16_t* out, cudaStream_t stream) {
    if (T < 0 || k < 1 || k > 8 || d % 8 != 0 || !y || !pos || !weight || !resid || !out) return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (k <= 2)
        return launch_pdl(combine_kernel<2>, dim3(static_cast<unsigned>(T)), dim3(kRowThreads), 0, stream, y, pos,
                          weight, resid, T, k, d, out);
    return launch_pdl(combine_kernel<8>, dim3(static_cast<unsigned>(T)), dim3(kRowThreads), 0, stream, y, pos, weight,
                      resid, T, k, d, out);
}

extern "C" int kl_combine_deferred(const float* y_part, int splits, int64_t split_rows, const int32_t* pos,
                                   const float* weight, const uint16_t* resid, int64_t T, int k, int d, uint16_t* out,
                                   cudaStream_t stream) {
    if (T < 0 || k < 1 || k > 8 || d % 8 != 0 || splits < 1 || splits > 4 || split_rows < 0 || !y_part || !pos ||
        !weight || !resid || !out)
        return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int64_t se = split_rows * d;
    if (k <= 2)
        return launch_pdl(combine_deferred_kernel<2>, dim3(static_cast<unsigned>(T)), dim3(kRowThreads), 0, stream,
                          y_part, splits, se, pos, weight, resid, T, k, d, out);
    return launch_pdl(combine_deferred_kernel<8>, dim3(static_cast<unsigned>(T)), dim3(kRowThreads), 0, stream, y_part,
                      splits, se, pos, weight, resid, T, k, d, out);
}

extern "C" int kl_coact_update(const int32_t* prev, const int32_t* cur, int64_t T, int k, int E, int layer,
                               int64_t* table, int64_t* marginal, cudaStream_t stream) {
    if (T < 0 || k < 1 || E < 1 || E > 64 || layer < 0 || !cur) return KL_EINVAL;
    if (layer == 0 ? marginal == nullptr : (table == nullptr || prev == nullptr)) return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int cells = layer == 0 ? E : E * E;
    const int blocks = static_cast<int>(T / 256 + 1 < 148 ? T / 256 + 1 : 148);
    if (int rc_ = launch_pdl(coact_kernel, dim3(blocks), dim3(256), cells * sizeof(int32_t), stream, prev, cur, T, k, E, layer, table, marginal)) return rc_;
    return check_launch();
}

extern "C" int kl_predict_scores(const int32_t* hist, const int64_t* table, int E, int layer, int64_t* score,
                                 cudaStream_t stream) {
    if (E < 1 || E > 1024 || layer < 1 || !hist || !table || !score) return KL_EINVAL;
    if (int rc_ = launch_pdl(predict_kernel, dim3(1), dim3(E < 32 ? 32 : E), 0, stream, hist, table, E, layer, score)) return rc_;
    return check_launch();
}

extern "C" int kl_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, float std_dev, cudaStream_t stream) {
    if (n < 0 || (n > 0 && dst == nullptr)) return KL_EINVAL;
    if (n == 0) return KL_OK;
    const int64_t blocks = (n + 255) / 256;
    fill_normal_kernel<<<static_cast<int>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, stream>>>(dst, n, seed,
                                                                                                      std_dev);
    return check_launch();
}

extern "C" int kl_route_override(const int32_t* forced, const float* logits, int T, int E, int k, int32_t* idx,
                                 float* weight, int32_t* hist, int32_t* first_pos, cudaStream_t stream) {
    if (T < 0 || E < 1 || k < 1 || k > 8 || !forced || !logits || !idx || !weight) return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (int rc_ = launch_pdl(route_override_kernel, dim3((T + 127) / 128), dim3(128), 0, stream, forced, logits, T, E, k, idx, weight, hist, first_pos)) return rc_;
    return check_launch();
}

extern "C" int kl_embed(const int32_t* ids, const uint16_t* table, int64_t T, int d, uint16_t* out,
                        cudaStream_t stream) {
    if (T < 0 || d % 8 != 0 || !ids || !table || !out) return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (int rc_ = launch_pdl(embed_kernel, dim3(grid_for(T, kWarpsPerBlock)), dim3(kWarpsPerBlock * 32), 0, stream, ids, table, T, d, out)) return rc_;
    return check_launch();
}

extern "C" int kl_argmax_bf16(const uint16_t* logits, int64_t T, int V, int32_t* out, cudaStream_t stream) {
    if (T < 0 || V < 1 || !logits || !out) return KL_EINVAL;
    if (T == 0) return KL_OK;
    if (int rc_ = launch_pdl(argmax_kernel, dim3(grid_for(T, kWarpsPerBlock)), dim3(kWarpsPerBlock * 32), 0, stream, logits, T, V, out)) return rc_;
    return check_launch();
}

// ---------------------------------------------------------------- EP helpers --
namespace kl {
namespace {

__global__ void map_ids_kernel(const int32_t* __restrict__ in, int64_t n, const int32_t* __restrict__ map,
                               int32_t* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = map[in[i]];
}

__global__ void sum_rows_i32_kernel(const int32_t* __restrict__ in, int rows, int cols, int32_t* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    int32_t s = 0;
    for (int r = 0; r < rows; ++r) s += in[static_cast<int64_t>(r) * cols + c];
    out[c] = s;
}

__global__ void add_i64_kernel(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

}  // namespace
}  // namespace kl

extern "C" int kl_map_ids(const int32_t* in, int64_t n, const int32_t* map, int32_t* out, cudaStream_t stream) {
    if (n < 0 || (n > 0 && (!in || !map || !out))) return KL_EINVAL;
    if (n == 0) return KL_OK;
    kl::map_ids_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, stream>>>(in, n, map, out);
    return kl::check_launch();
}

extern "C" int kl_sum_rows_i32(const int32_t* in, int rows, int cols, int32_t* out, cudaStream_t stream) {
    if (rows < 0 || cols < 1 || !in || !out) return KL_EINVAL;
    kl::sum_rows_i32_kernel<<<(cols + 127) / 128, 128, 0, stream>>>(in, rows, cols, out);
    return kl::check_launch();
}

extern "C" int kl_add_i64(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t stream) {
    if (n < 0 || (n > 0 && (!dst || !src))) return KL_EINVAL;
    if (n == 0) return KL_OK;
    kl::add_i64_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, stream>>>(dst, src, n);
    return kl::check_launch();
}
