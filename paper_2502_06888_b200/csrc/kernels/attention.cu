// SPDX-License-Identifier: Apache-2.0
// K6: attention pieces for compute_attention (reference schedule.cpp:313-338,
// priced as token_count * attn_per_token in simulator.cpp:15). The reference
// models KV retention only as a cache-size cap (model.hpp:60-73,
// KvRetentionPolicy::retained); here it is executed: each sequence keeps
// `sink` leading positions plus a ring of `cap - sink` most recent ones, and
// attention reads exactly the retained slots.
//
// Decode attention is HBM-bound (K and V of the retained slots are read once
// per (token, kv head); query heads of one GQA group share the reads through
// L1): algorithmic bytes per (sequence, layer) = retained * Hkv*hd*2 * 2.
#include <cstdint>

#include "common.cuh"

namespace kl {
namespace {

__device__ __forceinline__ int slot_of(int p, int cap, int sink) {
    return p < sink ? p : sink + (p - sink) % (cap - sink);
}

// qkv row layout: [Hq*hd | Hkv*hd | Hkv*hd]. One thread per (token, head, pair).
__global__ void rope_append_kernel(uint16_t* __restrict__ qkv, int64_t T, int Hq, int Hkv, int hd,
                                   const int32_t* __restrict__ pos, const int32_t* __restrict__ seq, float theta,
                                   uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int cap, int sink,
                                   int chunk_last_pos) {
    const int half = hd / 2;
    const int heads = Hq + Hkv;
    const int64_t per_tok = static_cast<int64_t>(heads) * half + static_cast<int64_t>(Hkv) * half;
    const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= T * per_tok) return;
    const int64_t t = id / per_tok;
    int64_t rem = id % per_tok;
    const int64_t width = static_cast<int64_t>(Hq + 2 * Hkv) * hd;
    uint16_t* row = qkv + t * width;
    const int p = pos[t];
    const int slot = slot_of(p, cap, sink);
    const bool to_cache = chunk_last_pos < 0 || p < sink || p > chunk_last_pos - (cap - sink);
    const int64_t cache_row = (static_cast<int64_t>(seq[t]) * cap + slot) * Hkv * hd;
    if (rem < static_cast<int64_t>(heads) * half) {
        const int head = static_cast<int>(rem / half);
        const int i = static_cast<int>(rem % half);
        const float inv = powf(theta, -2.0f * static_cast<float>(i) / static_cast<float>(hd));
        float sn, cs;
        sincosf(static_cast<float>(p) * inv, &sn, &cs);
        uint16_t* base = row + static_cast<int64_t>(head) * hd;
        const float a = bf2f(base[i]), b = bf2f(base[i + half]);
        const uint16_t ra = f2bf(a * cs - b * sn);
        const uint16_t rb = f2bf(b * cs + a * sn);
        base[i] = ra;
        base[i + half] = rb;
        if (head >= Hq && to_cache) {  // rotated key -> cache
            uint16_t* dst = kc + cache_row + static_cast<int64_t>(head - Hq) * hd;
            dst[i] = ra;
            dst[i + half] = rb;
        }
    } else {
        rem -= static_cast<int64_t>(heads) * half;
        if (!to_cache) return;
        const int kvh = static_cast<int>(rem / half);
        const int i = static_cast<int>(rem % half);
        const uint16_t* src = row + static_cast<int64_t>(Hq + Hkv + kvh) * hd;
        uint16_t* dst = vc + cache_row + static_cast<int64_t>(kvh) * hd;
        dst[i] = src[i];
        dst[i + half] = src[i + half];
    }
}

// One CTA (4 warps) per (token, kv head) covering the G query heads of the
// GQA group, so each retained K/V row is read from HBM exactly once:
//   1. thread-per-slot scores for all G heads (q in smem, broadcast reads);
//   2. per-head softmax (warp per head);
//   3. P.V with warps splitting the slots and lanes owning HD/32 dims each,
//      then a fixed-order cross-warp sum in smem.
constexpr int kAttnWarps = 4;

template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_decode_kernel(const uint16_t* __restrict__ q, int64_t q_stride, const int32_t* __restrict__ pos,
                   const int32_t* __restrict__ seq, int Hq, int Hkv, const uint16_t* __restrict__ kc,
                   const uint16_t* __restrict__ vc, int cap, int sink, float scale, uint16_t* __restrict__ out) {
    constexpr int PER = HD / 32;  // head dims owned by one lane in the P.V phase
    constexpr int GMAX = 8;
    extern __shared__ float smem_f[];
    const int G = Hq / Hkv;
    float* qs = smem_f;                     // [G][HD]
    float* sc = qs + G * HD;                // [G][cap]
    float* red = sc + G * cap;              // [warps][G][HD]
    float* inv_sum = red + kAttnWarps * G * HD;  // [G]
    const int t = blockIdx.x;
    const int kvh = blockIdx.y;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = pos[t];
    const int n = p + 1 < cap ? p + 1 : cap;  // retained slots (all valid)
    const int64_t row_stride = static_cast<int64_t>(Hkv) * HD;
    const uint16_t* kbase = kc + static_cast<int64_t>(seq[t]) * cap * row_stride + static_cast<int64_t>(kvh) * HD;
    const uint16_t* vbase = vc + static_cast<int64_t>(seq[t]) * cap * row_stride + static_cast<int64_t>(kvh) * HD;

    const uint16_t* qp = q + static_cast<int64_t>(t) * q_stride + static_cast<int64_t>(kvh) * G * HD;
    for (int i = threadIdx.x; i < G * HD; i += blockDim.x) qs[i] = bf2f(qp[i]) * scale;
    __syncthreads();

    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const uint16_t* kp = kbase + static_cast<int64_t>(j) * row_stride;
        float acc[GMAX];
#pragma unroll
        for (int g = 0; g < GMAX; ++g) acc[g] = 0.f;
#pragma unroll 4
        for (int c = 0; c < HD; c += 8) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(kp + c));
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            float kv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                kv[2 * i] = bf2f(static_cast<uint16_t>(ws[i] & 0xffffu));
                kv[2 * i + 1] = bf2f(static_cast<uint16_t>(ws[i] >> 16));
            }
#pragma unroll
            for (int g = 0; g < GMAX; ++g) {
                if (g < G) {
                    const float4 q0 = *reinterpret_cast<const float4*>(qs + g * HD + c);
                    const float4 q1 = *reinterpret_cast<const float4*>(qs + g * HD + c + 4);
                    acc[g] = fmaf(q0.x, kv[0], acc[g]);
                    acc[g] = fmaf(q0.y, kv[1], acc[g]);
                    acc[g] = fmaf(q0.z, kv[2], acc[g]);
                    acc[g] = fmaf(q0.w, kv[3], acc[g]);
                    acc[g] = fmaf(q1.x, kv[4], acc[g]);
                    acc[g] = fmaf(q1.y, kv[5], acc[g]);
                    acc[g] = fmaf(q1.z, kv[6], acc[g]);
                    acc[g] = fmaf(q1.w, kv[7], acc[g]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < GMAX; ++g)
            if (g < G) sc[g * cap + j] = acc[g];
    }
    __syncthreads();

    for (int g = wid; g < G; g += kAttnWarps) {
        float* s = sc + g * cap;
        float mx = -INFINITY;
        for (int j = lane; j < n; j += 32) mx = fmaxf(mx, s[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.f;
        for (int j = lane; j < n; j += 32) {
            const float e = __expf(s[j] - mx);
            s[j] = e;
            sum += e;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) inv_sum[g] = 1.0f / sum;
    }
    __syncthreads();

    float o[GMAX][PER];
#pragma unroll
    for (int g = 0; g < GMAX; ++g)
#pragma unroll
        for (int i = 0; i < PER; ++i) o[g][i] = 0.f;
    const int chunk = (n + kAttnWarps - 1) / kAttnWarps;
    const int j0 = wid * chunk, j1 = min(n, j0 + chunk);
    // Four V rows in flight per iteration (the loop is otherwise a serial
    // chain of dependent-latency loads).
    constexpr int U = 4;
    for (int jb = j0; jb < j1; jb += U) {
        float vv[U][PER];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = jb + u < j1 ? jb + u : j1 - 1;
            const uint16_t* vp = vbase + static_cast<int64_t>(j) * row_stride + lane * PER;
#pragma unroll
            for (int i = 0; i < PER; i += 2) {
                const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(vp + i));
                vv[u][i] = bf2f(static_cast<uint16_t>(w & 0xffffu));
                vv[u][i + 1] = bf2f(static_cast<uint16_t>(w >> 16));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (jb + u >= j1) break;
#pragma unroll
            for (int g = 0; g < GMAX; ++g) {
                if (g < G) {
                    const float pj = sc[g * cap + jb + u];
#pragma unroll
                    for (int i = 0; i < PER; ++i) o[g][i] = fmaf(pj, vv[u][i], o[g][i]);
                }
            }
        }
    }
#pragma unroll
    for (int g = 0; g < GMAX; ++g)
        if (g < G)
#pragma unroll
            for (int i = 0; i < PER; ++i) red[(wid * G + g) * HD + lane * PER + i] = o[g][i];
    __syncthreads();
    uint16_t* op = out + static_cast<int64_t>(t) * Hq * HD + static_cast<int64_t>(kvh) * G * HD;
    for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) acc += red[w * G * HD + i];
        op[i] = f2bf(acc * inv_sum[i / HD]);
    }
}

// Prefill: one warp per (query row, q head); keys from the same chunk's qkv
// rows; causal with sink + sliding-window retention; online softmax.
template <int HD>
__global__ void attn_prefill_kernel(const uint16_t* __restrict__ qkv, int n_seq, int L, int Hq, int Hkv, int cap,
                                    int sink, float scale, uint16_t* __restrict__ out) {
    constexpr int PER = HD / 32;
    const int64_t wid = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t rows = static_cast<int64_t>(n_seq) * L;
    if (wid >= rows * Hq) return;
    const int64_t row = wid / Hq;
    const int qh = static_cast<int>(wid % Hq);
    const int sq = static_cast<int>(row / L), i = static_cast<int>(row % L);
    const int kvh = qh / (Hq / Hkv);
    const int64_t width = static_cast<int64_t>(Hq + 2 * Hkv) * HD;
    const uint16_t* qp = qkv + row * width + static_cast<int64_t>(qh) * HD + lane * PER;
    float qv[PER], o[PER];
#pragma unroll
    for (int x = 0; x < PER; ++x) {
        qv[x] = bf2f(qp[x]) * scale;
        o[x] = 0.f;
    }
    const int window = cap - sink;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j <= i; ++j) {
        const bool kept = j < sink || j > i - window;
        if (!kept) continue;
        const int64_t krow = (static_cast<int64_t>(sq) * L + j) * width;
        const uint16_t* kp = qkv + krow + static_cast<int64_t>(Hq + kvh) * HD + lane * PER;
        const uint16_t* vp = qkv + krow + static_cast<int64_t>(Hq + Hkv + kvh) * HD + lane * PER;
        float dot = 0.f;
#pragma unroll
        for (int x = 0; x < PER; ++x) dot = fmaf(qv[x], bf2f(kp[x]), dot);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        const float nm = fmaxf(m, dot);
        const float corr = __expf(m - nm), pj = __expf(dot - nm);
#pragma unroll
        for (int x = 0; x < PER; ++x) o[x] = o[x] * corr + pj * bf2f(vp[x]);
        l = l * corr + pj;
        m = nm;
    }
    const float inv = 1.0f / l;
    uint16_t* op = out + row * Hq * HD + static_cast<int64_t>(qh) * HD + lane * PER;
#pragma unroll
    for (int x = 0; x < PER; ++x) op[x] = f2bf(o[x] * inv);
}

}  // namespace
}  // namespace kl

using namespace kl;

extern "C" int kl_rope_kv_append(uint16_t* qkv, int64_t T, int Hq, int Hkv, int hd, const int32_t* pos,
                                 const int32_t* seq, float rope_theta, uint16_t* k_cache, uint16_t* v_cache, int cap,
                                 int sink, int chunk_last_pos, cudaStream_t stream) {
    if (T < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || hd % 2 || cap <= sink || sink < 0) return KL_EINVAL;
    if (!qkv || !pos || !seq || !k_cache || !v_cache) return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int64_t n = T * ((static_cast<int64_t>(Hq) + 2 * Hkv) * (hd / 2));
    rope_append_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, stream>>>(qkv, T, Hq, Hkv, hd, pos, seq,
                                                                               rope_theta, k_cache, v_cache, cap, sink,
                                                                               chunk_last_pos);
    return check_launch();
}

extern "C" int kl_attn_decode(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq, int64_t T,
                              int Hq, int Hkv, int hd, const uint16_t* k_cache, const uint16_t* v_cache, int cap,
                              int sink, float scale, uint16_t* out, cudaStream_t stream) {
    if (hd != 128 && hd != 64) return KL_EUNSUPPORTED;
    if (T < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || Hq / Hkv > 32 || cap <= sink || !q || !pos || !seq || !out)
        return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int G = Hq / Hkv;
    if (G > 8) return KL_EUNSUPPORTED;
    const size_t smem = (static_cast<size_t>(G) * hd + static_cast<size_t>(G) * cap +
                         static_cast<size_t>(kAttnWarps) * G * hd + G) * sizeof(float);
    if (smem > 200 * 1024) return KL_EUNSUPPORTED;
    auto kern = hd == 128 ? attn_decode_kernel<128> : attn_decode_kernel<64>;
    if (smem > 48 * 1024)
        KL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<dim3(static_cast<unsigned>(T), Hkv), kAttnWarps * 32, smem, stream>>>(q, q_stride, pos, seq, Hq, Hkv,
                                                                               k_cache, v_cache, cap, sink, scale, out);
    return check_launch();
}

extern "C" int kl_attn_prefill(const uint16_t* qkv, int n_seq, int L, int Hq, int Hkv, int hd, int cap, int sink,
                               float scale, uint16_t* out, cudaStream_t stream) {
    if (hd != 128 && hd != 64) return KL_EUNSUPPORTED;
    if (n_seq < 0 || L < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || cap <= sink || !qkv || !out) return KL_EINVAL;
    const int64_t warps = static_cast<int64_t>(n_seq) * L * Hq;
    if (warps == 0) return KL_OK;
    auto kern = hd == 128 ? attn_prefill_kernel<128> : attn_prefill_kernel<64>;
    kern<<<static_cast<int>((warps + 7) / 8), 256, 0, stream>>>(qkv, n_seq, L, Hq, Hkv, cap, sink, scale, out);
    return check_launch();
}
