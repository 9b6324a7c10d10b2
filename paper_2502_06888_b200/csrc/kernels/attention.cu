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
#include <atomic>
#include <cstdint>
#include <mutex>
#include <cstdlib>

#include "common.cuh"
#include "tma_host.cuh"

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
    pdl_enter();
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
        float sn, cs;
        rope_cs(p, i, hd, theta, cs, sn);
        uint16_t* base = row + static_cast<int64_t>(head) * hd;
        const float a = bf2f(base[i]), b = bf2f(base[i + half]);
        const uint16_t ra = f2bf(rope_lo(a, b, cs, sn));
        const uint16_t rb = f2bf(rope_hi(a, b, cs, sn));
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

// rope_append_kernel over a QKV projection left as S fp32 split partials
// (kl_gemm_bf16_deferred): each element is first summed in the owner's order
// (own split S-1, then 0..S-2) and rounded to bf16 -- the value the GEMM's
// fixup would have stored -- then rotated / appended exactly as
// rope_append_kernel, and the full qkv row is written.
__device__ __forceinline__ float sum_split_elem(const float* __restrict__ part, int S, int64_t se, int64_t off) {
    float v = part[static_cast<int64_t>(S - 1) * se + off];
    for (int sp = 0; sp < S - 1; ++sp) v = __fadd_rn(v, part[sp * se + off]);
    return bf2f(f2bf(v));
}

// Four pairs per thread: float4 loads of each split's partials (the same
// sums and roundings as the scalar form).
__device__ __forceinline__ float4 sum_split_vec4(const float* __restrict__ part, int S, int64_t se, int64_t off) {
    float4 v = __ldg(reinterpret_cast<const float4*>(part + static_cast<int64_t>(S - 1) * se + off));
    for (int sp = 0; sp < S - 1; ++sp) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(part + sp * se + off));
        v.x = __fadd_rn(v.x, q.x);
        v.y = __fadd_rn(v.y, q.y);
        v.z = __fadd_rn(v.z, q.z);
        v.w = __fadd_rn(v.w, q.w);
    }
    return make_float4(bf2f(f2bf(v.x)), bf2f(f2bf(v.y)), bf2f(f2bf(v.z)), bf2f(f2bf(v.w)));
}

// Both halves of a rotation pair (offsets oa, ob) summed as sum_split_vec4
// does; for S <= 4 every split's loads are issued before the first add (one
// memory latency instead of a chain of S).
__device__ __forceinline__ void sum_split_pair4(const float* __restrict__ part, int S, int64_t se, int64_t oa,
                                                int64_t ob, float4& a, float4& b) {
    if (S > 4) {
        a = sum_split_vec4(part, S, se, oa);
        b = sum_split_vec4(part, S, se, ob);
        return;
    }
    float4 qa[4], qb[4];
#pragma unroll
    for (int sl = 0; sl < 4; ++sl)
        if (sl < S) {
            const int64_t sp = sl == 0 ? S - 1 : sl - 1;  // the owner's split first, then 0..S-2
            qa[sl] = __ldg(reinterpret_cast<const float4*>(part + sp * se + oa));
            qb[sl] = __ldg(reinterpret_cast<const float4*>(part + sp * se + ob));
        }
    float4 va = qa[0], vb = qb[0];
#pragma unroll
    for (int sl = 1; sl < 4; ++sl)
        if (sl < S) {
            va.x = __fadd_rn(va.x, qa[sl].x); va.y = __fadd_rn(va.y, qa[sl].y);
            va.z = __fadd_rn(va.z, qa[sl].z); va.w = __fadd_rn(va.w, qa[sl].w);
            vb.x = __fadd_rn(vb.x, qb[sl].x); vb.y = __fadd_rn(vb.y, qb[sl].y);
            vb.z = __fadd_rn(vb.z, qb[sl].z); vb.w = __fadd_rn(vb.w, qb[sl].w);
        }
    a = make_float4(bf2f(f2bf(va.x)), bf2f(f2bf(va.y)), bf2f(f2bf(va.z)), bf2f(f2bf(va.w)));
    b = make_float4(bf2f(f2bf(vb.x)), bf2f(f2bf(vb.y)), bf2f(f2bf(vb.z)), bf2f(f2bf(vb.w)));
}

__global__ void rope_append_deferred_vec_kernel(const float* __restrict__ part, int S, int64_t split_elems,
                                                uint16_t* __restrict__ qkv, int64_t T, int Hq, int Hkv, int hd,
                                                const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
                                                float theta, uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                                int cap, int sink, int chunk_last_pos) {
    pdl_enter();
    const int half = hd / 2, q4 = half / 4;
    const int heads = Hq + Hkv;
    const int64_t per_tok = static_cast<int64_t>(heads + Hkv) * q4;
    const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= T * per_tok) return;
    const int64_t t = id / per_tok;
    const int unit = static_cast<int>(id % per_tok);
    const int64_t width = static_cast<int64_t>(Hq + 2 * Hkv) * hd;
    uint16_t* row = qkv + t * width;
    const int64_t prow = t * width;
    const int p = pos[t];
    const bool to_cache = chunk_last_pos < 0 || p < sink || p > chunk_last_pos - (cap - sink);
    const int64_t cache_row = (static_cast<int64_t>(seq[t]) * cap + slot_of(p, cap, sink)) * Hkv * hd;
    const int head = unit / q4, i0 = (unit % q4) * 4;  // head in [0, Hq + 2 Hkv)
    const int64_t b0 = prow + static_cast<int64_t>(head) * hd;
    float4 a4, b4;
    sum_split_pair4(part, S, split_elems, b0 + i0, b0 + i0 + half, a4, b4);
    uint16_t ra[4], rb[4];
    if (head < heads) {
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float sn, cs;
            rope_cs(p, i0 + e, hd, theta, cs, sn);
            ra[e] = f2bf(rope_lo(av[e], bv[e], cs, sn));
            rb[e] = f2bf(rope_hi(av[e], bv[e], cs, sn));
        }
    } else {
        ra[0] = f2bf(a4.x); ra[1] = f2bf(a4.y); ra[2] = f2bf(a4.z); ra[3] = f2bf(a4.w);
        rb[0] = f2bf(b4.x); rb[1] = f2bf(b4.y); rb[2] = f2bf(b4.z); rb[3] = f2bf(b4.w);
    }
    const uint2 lo = make_uint2(static_cast<uint32_t>(ra[0]) | (static_cast<uint32_t>(ra[1]) << 16),
                                static_cast<uint32_t>(ra[2]) | (static_cast<uint32_t>(ra[3]) << 16));
    const uint2 hi = make_uint2(static_cast<uint32_t>(rb[0]) | (static_cast<uint32_t>(rb[1]) << 16),
                                static_cast<uint32_t>(rb[2]) | (static_cast<uint32_t>(rb[3]) << 16));
    uint16_t* base = row + static_cast<int64_t>(head) * hd;
    *reinterpret_cast<uint2*>(base + i0) = lo;
    *reinterpret_cast<uint2*>(base + i0 + half) = hi;
    if (head < Hq || !to_cache) return;
    uint16_t* dst = head < heads ? kc + cache_row + static_cast<int64_t>(head - Hq) * hd
                                 : vc + cache_row + static_cast<int64_t>(head - heads) * hd;
    *reinterpret_cast<uint2*>(dst + i0) = lo;
    *reinterpret_cast<uint2*>(dst + i0 + half) = hi;
}

__global__ void rope_append_deferred_kernel(const float* __restrict__ part, int S, int64_t split_elems,
                                            uint16_t* __restrict__ qkv, int64_t T, int Hq, int Hkv, int hd,
                                            const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
                                            float theta, uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                            int cap, int sink, int chunk_last_pos) {
    pdl_enter();
    const int half = hd / 2;
    const int heads = Hq + Hkv;
    const int64_t per_tok = static_cast<int64_t>(heads) * half + static_cast<int64_t>(Hkv) * half;
    const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= T * per_tok) return;
    const int64_t t = id / per_tok;
    int64_t rem = id % per_tok;
    const int64_t width = static_cast<int64_t>(Hq + 2 * Hkv) * hd;
    uint16_t* row = qkv + t * width;
    const int64_t prow = t * width;
    const int p = pos[t];
    const int slot = slot_of(p, cap, sink);
    const bool to_cache = chunk_last_pos < 0 || p < sink || p > chunk_last_pos - (cap - sink);
    const int64_t cache_row = (static_cast<int64_t>(seq[t]) * cap + slot) * Hkv * hd;
    if (rem < static_cast<int64_t>(heads) * half) {
        const int head = static_cast<int>(rem / half);
        const int i = static_cast<int>(rem % half);
        float sn, cs;
        rope_cs(p, i, hd, theta, cs, sn);
        const int64_t b0 = prow + static_cast<int64_t>(head) * hd;
        const float a = sum_split_elem(part, S, split_elems, b0 + i);
        const float b = sum_split_elem(part, S, split_elems, b0 + i + half);
        const uint16_t ra = f2bf(rope_lo(a, b, cs, sn));
        const uint16_t rb = f2bf(rope_hi(a, b, cs, sn));
        uint16_t* base = row + static_cast<int64_t>(head) * hd;
        base[i] = ra;
        base[i + half] = rb;
        if (head >= Hq && to_cache) {
            uint16_t* dst = kc + cache_row + static_cast<int64_t>(head - Hq) * hd;
            dst[i] = ra;
            dst[i + half] = rb;
        }
    } else {
        rem -= static_cast<int64_t>(heads) * half;
        const int kvh = static_cast<int>(rem / half);
        const int i = static_cast<int>(rem % half);
        const int64_t b0 = prow + static_cast<int64_t>(Hq + Hkv + kvh) * hd;
        const uint16_t v0 = f2bf(sum_split_elem(part, S, split_elems, b0 + i));
        const uint16_t v1 = f2bf(sum_split_elem(part, S, split_elems, b0 + i + half));
        uint16_t* src = row + static_cast<int64_t>(Hq + Hkv + kvh) * hd;
        src[i] = v0;
        src[i + half] = v1;
        if (!to_cache) return;
        uint16_t* dst = vc + cache_row + static_cast<int64_t>(kvh) * hd;
        dst[i] = v0;
        dst[i + half] = v1;
    }
}

// Token-per-block RoPE + KV append: the token's cos/sin table (hd/2 entries,
// the same powf / sincosf per element as rope_append_kernel, so results are
// bit-identical) is computed once into shared memory and shared by all
// Hq + Hkv rotated heads; each thread rotates two adjacent dims per step
// with 32-bit accesses; V rows are copied with 16-byte vectors.
constexpr int kRopeThreads = 256;
__global__ void __launch_bounds__(kRopeThreads)
rope_append_tok_kernel(uint16_t* __restrict__ qkv, int Hq, int Hkv, int hd, const int32_t* __restrict__ pos,
                       const int32_t* __restrict__ seq, float theta, uint16_t* __restrict__ kc,
                       uint16_t* __restrict__ vc, int cap, int sink, int chunk_last_pos) {
    pdl_enter();
    extern __shared__ float cs_tab[];  // [half] cos, then [half] sin
    const int half = hd / 2;
    const int64_t t = blockIdx.x;
    const int64_t width = static_cast<int64_t>(Hq + 2 * Hkv) * hd;
    uint16_t* row = qkv + t * width;
    const int p = pos[t];
    const int slot = slot_of(p, cap, sink);
    const bool to_cache = chunk_last_pos < 0 || p < sink || p > chunk_last_pos - (cap - sink);
    const int64_t cache_row = (static_cast<int64_t>(seq[t]) * cap + slot) * Hkv * hd;
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
        float sn, cs;
        rope_cs(p, i, hd, theta, cs, sn);
        cs_tab[i] = cs;
        cs_tab[half + i] = sn;
    }
    __syncthreads();
    const int pairs = half / 2;  // 2 dims per thread-step
    const int heads = Hq + Hkv;
    for (int w = threadIdx.x; w < heads * pairs; w += blockDim.x) {
        const int head = w / pairs, i = (w % pairs) * 2;
        uint16_t* base = row + static_cast<int64_t>(head) * hd;
        const uint32_t av = *reinterpret_cast<const uint32_t*>(base + i);
        const uint32_t bv = *reinterpret_cast<const uint32_t*>(base + i + half);
        uint16_t ra[2], rb[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const float a = bf2f(static_cast<uint16_t>(e ? av >> 16 : av & 0xffffu));
            const float b = bf2f(static_cast<uint16_t>(e ? bv >> 16 : bv & 0xffffu));
            const float cs = cs_tab[i + e], sn = cs_tab[half + i + e];
            ra[e] = f2bf(rope_lo(a, b, cs, sn));
            rb[e] = f2bf(rope_hi(a, b, cs, sn));
        }
        const uint32_t ro = static_cast<uint32_t>(ra[0]) | (static_cast<uint32_t>(ra[1]) << 16);
        const uint32_t rbo = static_cast<uint32_t>(rb[0]) | (static_cast<uint32_t>(rb[1]) << 16);
        *reinterpret_cast<uint32_t*>(base + i) = ro;
        *reinterpret_cast<uint32_t*>(base + i + half) = rbo;
        if (head >= Hq && to_cache) {  // rotated key -> cache
            uint16_t* dst = kc + cache_row + static_cast<int64_t>(head - Hq) * hd;
            *reinterpret_cast<uint32_t*>(dst + i) = ro;
            *reinterpret_cast<uint32_t*>(dst + i + half) = rbo;
        }
    }
    if (!to_cache) return;
    const uint4* vsrc = reinterpret_cast<const uint4*>(row + static_cast<int64_t>(Hq + Hkv) * hd);
    uint4* vdst = reinterpret_cast<uint4*>(vc + cache_row);
    for (int w = threadIdx.x; w < Hkv * hd / 8; w += blockDim.x) vdst[w] = vsrc[w];
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

// Split-KV decode ("flash-decoding"), the HBM-bound path: one CTA per
// (token, chunk of kDecChunk retained slots). The chunk's K and V rows of
// every KV head are contiguous in the cache ([seq][slot][Hkv][hd]), so one
// thread stages them with two 1D bulk copies (cp.async.bulk, full memory-
// level parallelism, no per-thread address math); scores start as soon as K
// lands while V is still in flight. Warps map to KV heads: lane = slot for
// q.k (rotated 16-byte reads, conflict-free), lane = head dims for p.V.
// Each CTA writes the chunk's unnormalised output with its running max and
// sum; attn_merge_kernel folds the chunks (fixed chunk order).
// Algorithmic bytes per (token, layer): retained * Hkv*hd*2 * 2.
constexpr int kDecChunk = 16;
constexpr int kDecThreads = 128;
constexpr int kKPad = 8;  // bf16 padding per staged K row: rows land 16 B apart in the banks

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int HD>
__global__ void __launch_bounds__(kDecThreads)
attn_decode_split_kernel(const uint16_t* __restrict__ q, int64_t q_stride, const int32_t* __restrict__ pos,
                         const int32_t* __restrict__ seq, int Hq, int Hkv, const uint16_t* __restrict__ kc,
                         const uint16_t* __restrict__ vc, int cap, float scale, float* __restrict__ part_o,
                         float* __restrict__ part_ml, int n_chunks) {
    constexpr int V8 = HD / 8;  // 16-byte vectors per head row
    extern __shared__ __align__(128) uint8_t dsm[];
    const int t = blockIdx.x, c = blockIdx.y;
    const int G = Hq / Hkv;
    const int row = Hkv * HD;        // elements per cache slot row (all KV heads)
    const int krow = row + kKPad;    // staged K row stride (padded)
    uint16_t* Ks = reinterpret_cast<uint16_t*>(dsm);
    uint16_t* Vs = Ks + kDecChunk * krow;
    float* qs = reinterpret_cast<float*>(Vs + kDecChunk * row);  // [Hq][HD], pre-scaled
    float* S = qs + Hq * HD;                                     // [Hq][kDecChunk]
    uint64_t* bars = reinterpret_cast<uint64_t*>(S + Hq * kDecChunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = min(pos[t] + 1, cap);
    const int j0 = c * kDecChunk;
    const int cnt = min(kDecChunk, n - j0);
    float* po = part_o + (static_cast<int64_t>(t) * n_chunks + c) * Hq * HD;
    float* pml = part_ml + (static_cast<int64_t>(t) * n_chunks + c) * Hq * 2;
    if (cnt <= 0) {
        for (int h = threadIdx.x; h < Hq; h += blockDim.x) {
            pml[2 * h] = -INFINITY;
            pml[2 * h + 1] = 0.f;
        }
        return;
    }
    const int64_t base = (static_cast<int64_t>(seq[t]) * cap + j0) * row;
    const uint32_t row_bytes = static_cast<uint32_t>(row) * 2;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(&bars[0], row_bytes * cnt);
        for (int j = 0; j < cnt; ++j) bulk_load(Ks + j * krow, kc + base + static_cast<int64_t>(j) * row, row_bytes, &bars[0]);
        mbar_arrive_expect_tx(&bars[1], row_bytes * cnt);
        bulk_load(Vs, vc + base, row_bytes * cnt, &bars[1]);
    }
    const uint16_t* qp = q + static_cast<int64_t>(t) * q_stride;
    for (int i = threadIdx.x; i < Hq * HD / 8; i += blockDim.x) {
        float v[8];
        const uint4 w = *reinterpret_cast<const uint4*>(qp + i * 8);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = bf2f(static_cast<uint16_t>(ws[k] & 0xffffu)) * scale;
            v[2 * k + 1] = bf2f(static_cast<uint16_t>(ws[k] >> 16)) * scale;
        }
        *reinterpret_cast<float4*>(qs + i * 8) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(qs + i * 8 + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
    __syncthreads();  // q staged; barrier inits visible
    mbar_wait(&bars[0], 0);

    // Scores: thread = (kv head h, slot j); every lane of a warp reads the
    // same q element (broadcast) and its own padded K row (no conflicts).
    for (int pr = threadIdx.x; pr < Hkv * kDecChunk; pr += blockDim.x) {
        const int h = pr / kDecChunk, j = pr % kDecChunk;
        if (j >= cnt) continue;
        const uint16_t* kr = Ks + j * krow + h * HD;
        float acc[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) acc[g] = 0.f;
#pragma unroll 4
        for (int x = 0; x < V8; ++x) {
            const uint4 w = *reinterpret_cast<const uint4*>(kr + x * 8);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            float kv[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                kv[2 * k] = bf2f(static_cast<uint16_t>(ws[k] & 0xffffu));
                kv[2 * k + 1] = bf2f(static_cast<uint16_t>(ws[k] >> 16));
            }
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                if (g < G) {
                    const float* qq = qs + (h * G + g) * HD + x * 8;
                    const float4 q0 = *reinterpret_cast<const float4*>(qq);
                    const float4 q1 = *reinterpret_cast<const float4*>(qq + 4);
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
        for (int g = 0; g < 8; ++g)
            if (g < G) S[(h * G + g) * kDecChunk + j] = acc[g];
    }
    __syncthreads();

    // Chunk softmax per q head: a half-warp per head, lane = slot.
    {
        const int half = lane >> 4, sl = lane & 15;
        for (int hq = warp * 2 + half; hq < Hq; hq += kDecThreads / 16) {
            const float sv = sl < cnt ? S[hq * kDecChunk + sl] : -INFINITY;
            float m = sv;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const float e = sl < cnt ? __expf(sv - m) : 0.f;
            float l = e;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
            S[hq * kDecChunk + sl] = e;
            if (sl == 0) {
                pml[2 * hq] = m;
                pml[2 * hq + 1] = l;
            }
        }
    }
    __syncthreads();
    mbar_wait(&bars[1], 0);

    // p.V: warp = kv head, lane owns HD/32 dims, G q heads.
    constexpr int PER = HD / 32;
    for (int h = warp; h < Hkv; h += kDecThreads / 32) {
        float o[8][PER];
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int i = 0; i < PER; ++i) o[g][i] = 0.f;
        for (int j = 0; j < cnt; ++j) {
            const uint16_t* vr = Vs + j * row + h * HD + lane * PER;
            float vv[PER];
            if constexpr (PER == 4) {
                const uint2 w = *reinterpret_cast<const uint2*>(vr);
                vv[0] = bf2f(static_cast<uint16_t>(w.x & 0xffffu));
                vv[1] = bf2f(static_cast<uint16_t>(w.x >> 16));
                vv[2] = bf2f(static_cast<uint16_t>(w.y & 0xffffu));
                vv[3] = bf2f(static_cast<uint16_t>(w.y >> 16));
            } else {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(vr);
                vv[0] = bf2f(static_cast<uint16_t>(w & 0xffffu));
                vv[1] = bf2f(static_cast<uint16_t>(w >> 16));
            }
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                if (g < G) {
                    const float pj = S[(h * G + g) * kDecChunk + j];
#pragma unroll
                    for (int i = 0; i < PER; ++i) o[g][i] = fmaf(pj, vv[i], o[g][i]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g < G) {
                float* dst = po + (h * G + g) * HD + lane * PER;
                if constexpr (PER == 4)
                    *reinterpret_cast<float4*>(dst) = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
                else
                    *reinterpret_cast<float2*>(dst) = make_float2(o[g][0], o[g][1]);
            }
        }
    }
}

// Fold the chunk partials of one (token, q head): fixed chunk order.
template <int HD>
__global__ void attn_merge_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml, int Hq,
                                  int n_chunks, uint16_t* __restrict__ out) {
    const int t = blockIdx.x, hq = blockIdx.y, d = threadIdx.x;
    const float* ml = part_ml + static_cast<int64_t>(t) * n_chunks * Hq * 2 + hq * 2;
    const float* po = part_o + static_cast<int64_t>(t) * n_chunks * Hq * HD + static_cast<int64_t>(hq) * HD + d;
    float M = -INFINITY;
#pragma unroll 8
    for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, ml[c * Hq * 2]);
    // Fixed-order fold; unrolled so the independent loads are in flight together.
    float L = 0.f, acc = 0.f;
#pragma unroll 8
    for (int c = 0; c < n_chunks; ++c) {
        const float m = ml[c * Hq * 2], l = ml[c * Hq * 2 + 1];
        if (m == -INFINITY) continue;  // empty chunk: its part_o was never written
        const float o = po[static_cast<int64_t>(c) * Hq * HD];
        const float w = __expf(m - M);
        L = fmaf(l, w, L);
        acc = fmaf(o, w, acc);
    }
    out[(static_cast<int64_t>(t) * Hq + hq) * HD + d] = f2bf(acc / L);
}

// ------------------------------------------ decode on mma.sync + TMA ring --
// Persistent split-KV decode. Work items are (token, KV-head group, chunk of
// kDmSlots retained slots), flattened token-major; CTA c owns the contiguous
// item range [c*I/C, (c+1)*I/C), so every SM streams the same number of K/V
// bytes. One producer thread stages each item's K and V with ONE 3D TMA load
// each (box = 16 slots x the group's HG*hd columns, 128B-swizzled with the
// slot as the swizzle row so ldmatrix over 8 slots is conflict-free; large
// copies are what reach HBM peak) plus, at the start of a segment, the
// token's q slice (1D bulk copy) into a kDmStages-deep ring. One consumer
// warp per KV head runs the item on the tensor cores (legacy HMMA m16n8k16):
// S = Q K^T with the G query heads of the GQA group as MMA rows, an online
// softmax on the accumulator fragments (the C fragment of S is the A
// fragment of P), O += P V with V through ldmatrix.trans. At the end of each
// (token, head group) segment the warp writes its unnormalised O with the
// running max (log2 domain) and sum; attn_merge_seg_kernel folds a token's
// segments in fixed chunk order.
// Algorithmic bytes per (token, layer): retained * Hkv*hd*2 * 2.
constexpr int kDmSlots = 16;
constexpr int kDmStages = 3;
constexpr int kDmMaxHG = 8;  // consumer warps (KV heads) per CTA
constexpr int kDmMaxG = 4;   // q heads folded per merge pass

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D += A B, m16n8k16, bf16 in, fp32 accumulate. A rows 8-15 are zero here.
__device__ __forceinline__ void hmma(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return static_cast<uint32_t>(f2bf(lo)) | (static_cast<uint32_t>(f2bf(hi)) << 16);
}
__device__ __forceinline__ void tma_load_3d_pol(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// Byte offset of (slot j, column col) in a staged box: 128-byte lines
// ordered (64-column chunk, slot), 16-byte units XOR-swizzled by slot % 8.
__device__ __forceinline__ uint32_t dm_off(int j, int col) {
    return static_cast<uint32_t>((((col >> 6) * kDmSlots + j) << 7) + ((((col >> 3) & 7) ^ (j & 7)) << 4));
}

// Fold the segment partials of the G q heads of one KV head of one token,
// in chunk order, with one warp. Lanes own chunks: the (max, sum) entries of
// all G heads load together; the segment starts ("live" chunks, max != -inf)
// are the same for every head, so each live chunk's G partial rows are
// gathered with independent loads before accumulating. Reads go through L2
// (ld.global.cg): the partials were written by other CTAs of this launch.
// ml: entry of (chunk 0, head 0), GH float2 per chunk; po: partial row of
// (chunk 0, head 0), HD floats per head; op: output row of head 0.
template <int HD>
__device__ __noinline__ void merge_heads_block(const float2* ml, const float* po, int G, int GH, int nv, uint16_t* op,
                                               int lane) {
    constexpr int PER = HD / 32;
    float M[kDmMaxG], L[kDmMaxG], acc[kDmMaxG][PER];
#pragma unroll
    for (int g = 0; g < kDmMaxG; ++g) {
        M[g] = -INFINITY;
        L[g] = 0.f;
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[g][i] = 0.f;
    }
    for (int k0 = 0; k0 < nv; k0 += 32) {
        const int k = k0 + lane;
#pragma unroll
        for (int g = 0; g < kDmMaxG; ++g)
            if (g < G && k < nv) M[g] = fmaxf(M[g], __ldcg(ml + static_cast<int64_t>(k) * GH + g).x);
    }
#pragma unroll
    for (int g = 0; g < kDmMaxG; ++g)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M[g] = fmaxf(M[g], __shfl_xor_sync(0xffffffffu, M[g], o));
    for (int k0 = 0; k0 < nv; k0 += 32) {
        const int k = k0 + lane;
        float2 e[kDmMaxG];
#pragma unroll
        for (int g = 0; g < kDmMaxG; ++g)
            e[g] = g < G && k < nv ? __ldcg(ml + static_cast<int64_t>(k) * GH + g) : make_float2(-INFINITY, 0.f);
        float w[kDmMaxG];
#pragma unroll
        for (int g = 0; g < kDmMaxG; ++g) {
            w[g] = e[g].x == -INFINITY ? 0.f : exp2f(e[g].x - M[g]);
            L[g] = fmaf(e[g].y, w[g], L[g]);
        }
        unsigned live = __ballot_sync(0xffffffffu, e[0].x != -INFINITY);
        while (live) {
            const int src = __ffs(live) - 1;
            live &= live - 1;
            const float* p = po + static_cast<int64_t>(k0 + src) * GH * HD + lane * PER;
            float v[kDmMaxG][PER];
#pragma unroll
            for (int g = 0; g < kDmMaxG; ++g) {
                if (g >= G) continue;
                if constexpr (PER == 4) {
                    const float4 x = __ldcg(reinterpret_cast<const float4*>(p + g * HD));
                    v[g][0] = x.x; v[g][1] = x.y; v[g][2] = x.z; v[g][3] = x.w;
                } else {
                    const float2 x = __ldcg(reinterpret_cast<const float2*>(p + g * HD));
                    v[g][0] = x.x; v[g][1] = x.y;
                }
            }
#pragma unroll
            for (int g = 0; g < kDmMaxG; ++g) {
                if (g >= G) continue;
                const float wg = __shfl_sync(0xffffffffu, w[g], src);
#pragma unroll
                for (int i = 0; i < PER; ++i) acc[g][i] = fmaf(v[g][i], wg, acc[g][i]);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < kDmMaxG; ++g) {
        if (g >= G) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L[g] += __shfl_xor_sync(0xffffffffu, L[g], o);
        const float inv = 1.f / L[g];
        uint16_t* o = op + static_cast<int64_t>(g) * HD + lane * PER;
        if constexpr (PER == 4)
            *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16(acc[g][0] * inv, acc[g][1] * inv),
                                                      pack_bf16(acc[g][2] * inv, acc[g][3] * inv));
        else
            *reinterpret_cast<uint32_t*>(o) = pack_bf16(acc[g][0] * inv, acc[g][1] * inv);
    }
}

// Up to kDmMaxG heads per pass (register arrays stay small); out of line so
// the rare merge does not raise the main loop's register pressure.
template <int HD>
__device__ __forceinline__ void merge_heads_warp(const float2* ml, const float* po, int G, int GH, int nv,
                                                 uint16_t* op, int lane) {
    for (int gb = 0; gb < G; gb += kDmMaxG)
        merge_heads_block<HD>(ml + gb, po + static_cast<int64_t>(gb) * HD, min(kDmMaxG, G - gb), GH, nv,
                              op + static_cast<int64_t>(gb) * HD, lane);
}

template <int HD>
__global__ void __launch_bounds__((kDmMaxHG + 1) * 32)
attn_decode_mma_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                       const uint16_t* __restrict__ q, int64_t q_stride, const int32_t* __restrict__ pos,
                       const int32_t* __restrict__ seq, int Hq, int Hkv, int HG, int cap, float scale_log2,
                       float* part_o, float* part_ml, int n_chunks, int64_t n_items, uint16_t* __restrict__ out,
                       unsigned long long* counters, uint32_t tag, int whole, int nst, int mode) {
    pdl_enter();
    const int G = Hq / Hkv, HGn = Hkv / HG;
    const uint32_t box_bytes = kDmSlots * HG * HD * 2;
    const int qelems = HG * G * HD;
    const uint32_t stage_bytes = (2 * box_bytes + qelems * 2 + 1023) & ~1023u;
    extern __shared__ uint8_t dsm_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(nst) * stage_bytes);
    uint64_t* empty = full + nst;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // whole: ranges cover whole (token, group) pairs, so no segment is split
    // across CTAs and every output is written directly.
    const int64_t pairs = n_items / n_chunks;
    const int64_t i0 = whole ? static_cast<int64_t>(blockIdx.x) * pairs / gridDim.x * n_chunks
                             : static_cast<int64_t>(blockIdx.x) * n_items / gridDim.x;
    const int64_t i1 = whole ? static_cast<int64_t>(blockIdx.x + 1) * pairs / gridDim.x * n_chunks
                             : static_cast<int64_t>(blockIdx.x + 1) * n_items / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], HG);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == HG) {  // producer
        if (lane != 0) return;
        const uint64_t kv_pol = l2_policy_evict_first();
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
        int64_t it = 0;
        int ps = 0;          // ring slot of the next item
        uint32_t pph = 0;    // its fill round parity
        // (token, group, chunk) of i0, then advanced incrementally; pos/seq
        // are read once per (token, group) segment.
        int k = static_cast<int>(i0 % n_chunks), hg = static_cast<int>((i0 / n_chunks) % HGn);
        int t = static_cast<int>(i0 / n_chunks / HGn);
        int n = min(pos[t] + 1, cap), row_t = seq[t] * cap;
        for (int64_t i = i0; i < i1; ++i, ++k) {
            if (k == n_chunks) {
                k = 0;
                if (++hg == HGn) {
                    hg = 0;
                    ++t;
                    n = min(pos[t] + 1, cap);
                    row_t = seq[t] * cap;
                }
            }
            const int j0 = k * kDmSlots;
            if (n - j0 <= 0) continue;
            const bool seg_first = i == i0 || k == 0;
            const int s = ps;
            if (it >= nst) mbar_wait(&empty[s], pph ^ 1u);
            if (++ps == nst) {
                ps = 0;
                pph ^= 1u;
            }
            uint8_t* st = ring + static_cast<size_t>(s) * stage_bytes;
            mbar_arrive_expect_tx(&full[s], 2 * box_bytes + (seg_first ? qelems * 2u : 0u));
            const int row = row_t + j0, chunk = hg * HG * HD / 64;
            if (mode & 4) {  // KV read once per step: L2 evict-first, so reused weights stay resident
                tma_load_3d_pol(st, &tmap_k, &full[s], 0, row, chunk, kv_pol);
                tma_load_3d_pol(st + box_bytes, &tmap_v, &full[s], 0, row, chunk, kv_pol);
            } else {
                tma_load_3d(st, &tmap_k, &full[s], 0, row, chunk);
                tma_load_3d(st + box_bytes, &tmap_v, &full[s], 0, row, chunk);
            }
            if (seg_first)
                bulk_load(st + 2 * box_bytes, q + static_cast<int64_t>(t) * q_stride + static_cast<int64_t>(hg) * HG * G * HD,
                          qelems * 2u, &full[s]);
            ++it;
        }
        return;
    }

    // Consumer warp = KV head `warp` of the group. Fragment roles: row g =
    // lane/4 is the query head within the GQA group (valid for g < G),
    // c4 = lane%4 picks the column pair.
    const int h = warp, g = lane >> 2, c4 = lane & 3;
    constexpr int KS = HD / 16, NT = HD / 8;
    uint32_t qa[KS][2];
    float o[NT][4];
    float m_run = -INFINITY, l_run = 0.f;
    bool seg_valid = false;
    int64_t seg_item = 0;
    int cs_ = 0;          // ring slot of the next item
    uint32_t cph = 0;     // its fill round parity
    int64_t it = 0;
    int k = static_cast<int>(i0 % n_chunks), hg = static_cast<int>((i0 / n_chunks) % HGn);
    int t = static_cast<int>(i0 / n_chunks / HGn);
    int n = min(pos[t] + 1, cap);
    for (int64_t i = i0; i < i1; ++i, ++k) {
        if (k == n_chunks) {
            k = 0;
            if (++hg == HGn) {
                hg = 0;
                n = min(pos[++t] + 1, cap);
            }
        }
        const int j0 = k * kDmSlots;
        const int cnt = min(kDmSlots, n - j0);
        const bool seg_first = i == i0 || k == 0;
        const bool seg_last = i == i1 - 1 || k == n_chunks - 1;
        if (seg_first) {
            seg_valid = cnt > 0;
            seg_item = i;
        }
        if (cnt > 0) {
            const int s = cs_;
            mbar_wait(&full[s], cph);
            if (++cs_ == nst) {
                cs_ = 0;
                cph ^= 1u;
            }
            uint8_t* Kb = ring + static_cast<size_t>(s) * stage_bytes;
            uint8_t* Vb = Kb + box_bytes;
            if ((mode & 3) >= 2) {  // load-only timing probe
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                ++it;
                continue;
            }
            if (seg_first) {
                const uint16_t* Qs = reinterpret_cast<const uint16_t*>(Kb + 2 * box_bytes) + (h * G + g) * HD + 2 * c4;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    qa[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(Qs + ks * 16) : 0u;
                    qa[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(Qs + ks * 16 + 8) : 0u;
                }
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
                m_run = -INFINITY;
                l_run = 0.f;
            }
            if (cnt < kDmSlots) {
                // Ragged chunk: rows past the retained count may be unwritten
                // cache memory; zero this head's V rows there (p = 0 must not
                // meet a NaN).
                constexpr int LINES = HD / 64;
                const int units = (kDmSlots - cnt) * LINES * 8;
                for (int u = lane; u < units; u += 32) {
                    const int j = cnt + u / (LINES * 8), line = (u / 8) % LINES, w = u & 7;
                    *reinterpret_cast<uint4*>(Vb + (((h * LINES + line) * kDmSlots + j) << 7) + (w << 4)) =
                        make_uint4(0u, 0u, 0u, 0u);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
            }
            // S = Q K^T over the chunk's 16 slots (two n-tiles of 8 slots).
            const uint32_t kb = smem_u32(Kb), vb = smem_u32(Vb);
            float sc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
                const int j = nt * 8 + (lane & 7);
#pragma unroll
                for (int kp = 0; kp < HD / 32; ++kp) {
                    uint32_t r0, r1, r2, r3;
                    ldsm_x4(kb + dm_off(j, h * HD + kp * 32 + (lane >> 3) * 8), r0, r1, r2, r3);
                    hmma(sc[nt], qa[2 * kp][0], qa[2 * kp][1], r0, r1);
                    hmma(sc[nt], qa[2 * kp + 1][0], qa[2 * kp + 1][1], r2, r3);
                }
            }
            // Online softmax on row g: this lane holds slots 2c4, 2c4+1, 8+2c4, 9+2c4.
            float x[4] = {sc[0][0], sc[0][1], sc[1][0], sc[1][1]};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int slot = (e >> 1) * 8 + 2 * c4 + (e & 1);
                x[e] = slot < cnt ? x[e] * scale_log2 : -INFINITY;
            }
            float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m_run, mx);
            const float m_use = m_new == -INFINITY ? 0.f : m_new;
            const float alpha = exp2f(m_run - m_use);
            float p[4], rs = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                p[e] = exp2f(x[e] - m_use);
                rs += p[e];
            }
            rs += __shfl_xor_sync(0xffffffffu, rs, 1);
            rs += __shfl_xor_sync(0xffffffffu, rs, 2);
            l_run = l_run * alpha + rs;
            m_run = m_new;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                o[nt][0] *= alpha;
                o[nt][1] *= alpha;
            }
            const uint32_t pa0 = pack_bf16(p[0], p[1]), pa2 = pack_bf16(p[2], p[3]);
            // O += P V: V^T fragments through ldmatrix.trans, 16 dims per x4.
            const int jv = ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
            for (int dp = 0; dp < HD / 16; ++dp) {
                uint32_t r0, r1, r2, r3;
                ldsm_x4_t(vb + dm_off(jv, h * HD + dp * 16 + (lane >> 4) * 8), r0, r1, r2, r3);
                hmma(o[2 * dp], pa0, pa2, r0, r1);
                hmma(o[2 * dp + 1], pa0, pa2, r2, r3);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            ++it;
            if (!seg_first && c4 == 0 && g < G) {  // not a segment start: nothing to fold here
                part_ml[(i * (HG * G) + h * G + g) * 2] = -INFINITY;
                part_ml[(i * (HG * G) + h * G + g) * 2 + 1] = 0.f;
            }
        }
        if (!seg_last) continue;
        if (seg_item == (static_cast<int64_t>(t) * HGn + hg) * n_chunks && k == n_chunks - 1) {
            // The whole (token, group) ran in this warp: normalise and store.
            if (g < G) {
                const float inv = 1.f / l_run;
                uint16_t* op = out + (static_cast<int64_t>(t) * Hq + (hg * HG + h) * G + g) * HD + 2 * c4;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    *reinterpret_cast<uint32_t*>(op + nt * 8) = pack_bf16(o[nt][0] * inv, o[nt][1] * inv);
            }
            continue;
        }
        if (seg_valid && g < G) {
            const int hq_local = h * G + g;
            float* po = part_o + (seg_item * (HG * G) + hq_local) * HD + 2 * c4;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<float2*>(po + nt * 8) = make_float2(o[nt][0], o[nt][1]);
            if (c4 == 0) {
                part_ml[(seg_item * (HG * G) + hq_local) * 2] = m_run;
                part_ml[(seg_item * (HG * G) + hq_local) * 2 + 1] = l_run;
            }
        }
        // Count this segment for its (token, KV head); the warp completing
        // the count folds the token's G q heads of this KV head (no merge
        // launch, no CTA-wide sync). The counter word is (tag << 32 | count):
        // a word left by any other use of the workspace never carries this
        // call's tag (a NaN pattern).
        __syncwarp();  // the lanes' partial writes are ordered before lane 0's release below
        const int64_t base = (static_cast<int64_t>(t) * HGn + hg) * n_chunks;
        unsigned last = 0;
        if (lane == 0) {
            const int64_t C = gridDim.x;
            auto cta_of = [&](int64_t x) { return ((x + 1) * C + n_items - 1) / n_items - 1; };
            const unsigned need = static_cast<unsigned>(cta_of(base + n_chunks - 1) - cta_of(base) + 1);
            unsigned long long* cp = counters + (static_cast<int64_t>(t) * Hkv + hg * HG + h);
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(cp), nxt;
            for (;;) {
                nxt = static_cast<uint32_t>(cur >> 32) == tag ? cur + 1 : (static_cast<unsigned long long>(tag) << 32) | 1ull;
                unsigned long long prev;
                // acq_rel at gpu scope: releases this warp's partials, and the
                // completing warp acquires every other contributor's.
                asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;"
                             : "=l"(prev) : "l"(cp), "l"(cur), "l"(nxt) : "memory");
                if (prev == cur) break;
                cur = prev;
            }
            last = static_cast<unsigned>(nxt & 0xffffffffull) == need;
            if (last) *reinterpret_cast<volatile unsigned long long*>(cp) = 0ull;
        }
        if (__shfl_sync(0xffffffffu, last, 0)) {
            const int GH = HG * G;
            merge_heads_warp<HD>(reinterpret_cast<const float2*>(part_ml) + base * GH + h * G,
                                 part_o + (base * GH + h * G) * HD, G, GH, (n + kDmSlots - 1) / kDmSlots,
                                 out + (static_cast<int64_t>(t) * Hq + hg * GH + h * G) * HD, lane);
        }
    }
}

// ------------------------------------------------ prefill on tcgen05 -------
// One CTA per (128/G query positions of one sequence, one KV head): the G
// query heads of the GQA group are stacked into the 128 MMA rows, so every
// K/V tile is shared by the whole group. Keys come in 128-row blocks that
// cover the causal sink + sliding window of the tile. Two passes, so the
// output needs no rescaling in TMEM:
//   pass 1: S = Q K^T (TMEM) per block -> row max and sum (thread = row);
//   pass 2: S again -> P = exp(S - max) / sum as bf16 into a 128B-swizzled
//           smem tile (the MMA's A operand) -> O += P V with V read
//           MN-major straight from its TMA tile (no transpose pass).
// Roofline: tensor-bound; FLOPs per (row, head, retained key) = 4 * hd.
constexpr int kPfThreads = 256;  // two warps per TMEM lane quarter, each owning half the key columns
constexpr int kPfParts = kPfThreads / 128;
constexpr int kPfKeys = 128;  // keys per block (MMA N for S, K for P.V)

// UMMA smem descriptor, MN-major operand in 128B-swizzled TMA tiles: 64
// elements (128 B) contiguous along MN, 8-row atoms of 1024 B along K;
// LBO = byte distance between 64-element MN chunks, SBO = 1024.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

template <int HD, int KEYS>
__global__ void __launch_bounds__(kPfThreads)
attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_kv,
                       int L, int Hq, int Hkv, int sink, int window, float scale, uint16_t* __restrict__ out) {
    constexpr int NCH = HD / 64;                  // 64-wide swizzle chunks along hd
    constexpr int kChunk = 128 * 128;             // bytes of a [128 rows x 64] bf16 tile (Q, P)
    constexpr int kBlk = NCH * kChunk;            // the Q tile
    constexpr int kvChunk = KEYS * 128;           // bytes of a [KEYS keys x 64] bf16 tile
    constexpr int kvBlk = NCH * kvChunk;          // one K (or V) block of KEYS keys
    constexpr int VBUF = KEYS == 64 ? 1 : 2;      // 64-key blocks: one V buffer, so 2 CTAs fit per SM
    constexpr int PCH = KEYS / 64;                // 64-key chunks of the P tile
    extern __shared__ uint8_t dsm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* Qs = sm;                       // NCH x [128 rows x 128 B]
    uint8_t* Kb = Qs + kBlk;                // 2 buffers: K blocks, prefetched one ahead
    uint8_t* Vb = Kb + 2 * kvBlk;           // VBUF buffers: V blocks
    uint8_t* Ps = Vb + VBUF * kvBlk;        // PCH x [128 rows x 128 B]  (keys 0-63, 64-127)
    uint64_t* bars = reinterpret_cast<uint64_t*>(Ps + PCH * kChunk);
    uint64_t* q_bar = &bars[0];
    uint64_t* k_bar = &bars[1];             // [2]
    uint64_t* v_bar = &bars[3];             // [2]
    uint64_t* s_bar = &bars[5];             // [2] S = QK^T done, per TMEM S buffer
    uint64_t* o_bar = &bars[7];             // O += PV done
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);

    const int G = Hq / Hkv;
    const int P = 128 / G;  // query positions per tile
    const int tile = blockIdx.x, kvh = blockIdx.y, sq = blockIdx.z;
    const int i0 = tile * P;
    const int64_t row0 = static_cast<int64_t>(sq) * L;
    const int r = threadIdx.x & 127;  // MMA row = TMEM lane
    const int half = threadIdx.x >> 7; // column part: keys [64*half, +64), O columns [HD/2*half, +HD/2)
    const int warp = threadIdx.x >> 5;
    const int g = r / P, i = i0 + r % P;
    float* stats = reinterpret_cast<float*>(tslot + 4);  // [parts][2][128] (m, l)

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_q);
        tma_prefetch_desc(&tmap_kv);
        for (int x = 0; x < 8; ++x) mbar_init(&bars[x], 1);
        mbar_fence_init();
    }
    constexpr uint32_t kTmemCols = 2 * KEYS + HD <= 256 ? 256 : 512;
    if (warp == 0) tmem_alloc(tslot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // Two S buffers (the next block's QK^T runs while this one's softmax is
    // computed) and O.
    const uint32_t tS0 = tmem, tO = tmem + 2 * KEYS;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;

    // Key blocks: [lo, hi] covering the window of the tile, plus block 0 for the sink.
    const int last = min(i0 + P - 1, L - 1);
    const int b_lo = max(0, i0 - window + 1) / KEYS, b_hi = last / KEYS;
    const bool sink_block = sink > 0 && b_lo > 0;
    const int nblk = (b_hi - b_lo + 1) + (sink_block ? 1 : 0);
    auto block_of = [&](int n) { return sink_block ? (n == 0 ? 0 : b_lo + n - 1) : b_lo + n; };

    const uint32_t idesc_s = idesc_bf16_f32(128, KEYS);
    const uint32_t idesc_o = idesc_bf16_f32(128, HD) | (1u << 16);  // B (V) MN-major

    // K loads form one sequence over both passes (index ki: pass 1 blocks
    // 0..nblk-1, then pass 2 again), V loads one over pass 2; each ring is two
    // buffers deep and issued one use ahead, so TMA latency hides behind the
    // previous block's MMA + softmax.
    const int k_total = 2 * nblk;
    auto load_k = [&](int ki) {  // thread 0
        const int bb = ki & 1;
        const int krow = static_cast<int>(row0 + block_of(ki % nblk) * KEYS);
        mbar_arrive_expect_tx(&k_bar[bb], kvBlk);
        for (int c = 0; c < NCH; ++c)
            tma_load_2d(Kb + bb * kvBlk + c * kvChunk, &tmap_kv, &k_bar[bb], (Hq + kvh) * HD + c * 64, krow);
    };
    auto load_v = [&](int vi) {
        const int bb = vi % VBUF;
        const int krow = static_cast<int>(row0 + block_of(vi) * KEYS);
        mbar_arrive_expect_tx(&v_bar[bb], kvBlk);
        for (int c = 0; c < NCH; ++c)
            tma_load_2d(Vb + bb * kvBlk + c * kvChunk, &tmap_kv, &v_bar[bb], (Hq + Hkv + kvh) * HD + c * 64, krow);
    };
    const bool leader = threadIdx.x == 0;
    if (leader) {
        mbar_arrive_expect_tx(q_bar, NCH * kChunk);
        for (int gg = 0; gg < G; ++gg)
            for (int c = 0; c < NCH; ++c)
                tma_load_2d(Qs + c * kChunk + gg * P * 128, &tmap_q, q_bar, (kvh * G + gg) * HD + c * 64,
                            static_cast<int>(row0 + i0));
        load_k(0);
        if (k_total > 1) load_k(1);
        load_v(0);
        if (VBUF == 2 && nblk > 1) load_v(1);
    }
    auto mma_s = [&](int ki) {  // thread 0: S buffer ki&1 = Q K^T for K load ki
        const int bb = ki & 1;
        mbar_wait(&k_bar[bb], (ki >> 1) & 1);
        tc_fence_after();
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                tc_mma_bf16(tS0 + bb * KEYS, sw128_kmajor_desc(smem_u32(Qs + c * kChunk) + k * 32),
                            sw128_kmajor_desc(smem_u32(Kb + bb * kvBlk + c * kvChunk) + k * 32), idesc_s, (c | k) != 0);
        tc_commit(&s_bar[bb]);
    };
    // S buffer b completes once per K load with that parity: load ki waits
    // phase (ki >> 1) & 1.
    auto wait_s = [&](int ki) {
        mbar_wait(&s_bar[ki & 1], (ki >> 1) & 1);
        __syncwarp();
        tc_fence_after();
    };
    auto valid = [&](int j) { return j <= i && j < L && (j < sink || j > i - window); };
    // A 32-key chunk is entirely retained for this row when its first key is
    // inside the window and its last is causal and in range.
    auto all_valid = [&](int j0) { return j0 > i - window && j0 + 31 <= i && j0 + 31 < L; };

    // Pass 1: row max and sum over the retained keys (each half its columns).
    float m = -INFINITY, l = 0.f;
    if (leader) {
        mbar_wait(q_bar, 0);
        mma_s(0);
    }
    for (int n = 0; n < nblk; ++n) {
        const int b = block_of(n);
        // Next block's (or pass 2's first) QK^T into the other S buffer, ahead
        // of this block's softmax; its K was loaded two uses back.
        if (leader && n + 1 < k_total) mma_s(n + 1);
        wait_s(n);
        if (leader && n + 2 < k_total) load_k(n + 2);  // its buffer's MMA has completed
        const uint32_t tS = tS0 + (n & 1) * KEYS;
        for (int c0 = half * (KEYS / kPfParts); c0 < (half + 1) * (KEYS / kPfParts); c0 += 32) {
            float v[32];
            tmem_ld32(tS + lane_off + c0, v);
            float bm = m;
            const int j0 = b * KEYS + c0;
            if (all_valid(j0)) {
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    v[x] *= scale;
                    bm = fmaxf(bm, v[x]);
                }
            } else {
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    v[x] = valid(j0 + x) ? v[x] * scale : -INFINITY;
                    bm = fmaxf(bm, v[x]);
                }
            }
            if (bm != -INFINITY) {  // (no divergent exit: the TMEM loads are warp-collective)
                float sum = 0.f;
#pragma unroll
                for (int x = 0; x < 32; ++x) sum += __expf(v[x] - bm);
                l = (m == -INFINITY ? 0.f : l * __expf(m - bm)) + sum;
                m = bm;
            }
        }
        tc_fence_before();
        __syncthreads();  // S buffer consumed
    }
    // Combine the two column halves' running (max, sum) per row.
    stats[(half * 2 + 0) * 128 + r] = m;
    stats[(half * 2 + 1) * 128 + r] = l;
    __syncthreads();
    {
        float mm = -INFINITY;
#pragma unroll
        for (int q = 0; q < kPfParts; ++q) mm = fmaxf(mm, stats[(q * 2) * 128 + r]);
        float ll = 0.f;
#pragma unroll
        for (int q = 0; q < kPfParts; ++q) {
            const float mq = stats[(q * 2) * 128 + r];
            if (mq != -INFINITY) ll += stats[(q * 2 + 1) * 128 + r] * __expf(mq - mm);
        }
        m = mm;
        l = ll;
    }
    const float inv_l = 1.0f / l;

    // Pass 2: P = softmax row (bf16, swizzled A tile), O += P V. The next
    // block's QK^T is issued before this block's P is built; the P tile is
    // rewritten only after the previous P.V completed.
    uint32_t o_phase = 0;
    for (int n = 0; n < nblk; ++n) {
        const int b = block_of(n);
        const int ki = nblk + n;
        if (leader && ki + 1 < k_total) mma_s(ki + 1);
        wait_s(ki);
        if (leader && ki + 2 < k_total) load_k(ki + 2);
        if (n > 0) {  // P.V(n-1) done: P reusable, its V buffer free
            mbar_wait(o_bar, o_phase);
            o_phase ^= 1;
            __syncwarp();
            tc_fence_after();
            if (leader && n - 1 + VBUF < nblk) load_v(n - 1 + VBUF);
        }
        const uint32_t tS = tS0 + (ki & 1) * KEYS;
        for (int c0 = half * (KEYS / kPfParts); c0 < (half + 1) * (KEYS / kPfParts); c0 += 32) {
            float v[32];
            tmem_ld32(tS + lane_off + c0, v);
            uint8_t* prow = Ps + (c0 / 64) * kChunk + r * 128;
            const int j0 = b * KEYS + c0;
            const bool full = all_valid(j0);
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
                uint32_t w[4];
#pragma unroll
                for (int h2 = 0; h2 < 4; ++h2) {
                    const int x0 = q8 * 8 + h2 * 2;
                    const int j = j0 + x0;
                    const float p0 = (full || valid(j)) ? __expf(v[x0] * scale - m) * inv_l : 0.f;
                    const float p1 = (full || valid(j + 1)) ? __expf(v[x0 + 1] * scale - m) * inv_l : 0.f;
                    w[h2] = pack2(p0, p1);
                }
                const int unit = ((c0 % 64) / 8 + q8) ^ (r & 7);  // 128B swizzle: 16-byte unit ^ row%8
                *reinterpret_cast<uint4*>(prow + unit * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        if (leader) {
            tc_fence_after();
            const int vb = n % VBUF;
            mbar_wait(&v_bar[vb], (n / VBUF) & 1);
            for (int kc = 0; kc < PCH; ++kc)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    tc_mma_bf16(tO, sw128_kmajor_desc(smem_u32(Ps + kc * kChunk) + k * 32),
                                sw128_mnmajor_desc(smem_u32(Vb + vb * kvBlk) + (kc * 64 + k * 16) * 128, kvChunk),
                                idesc_o, (n > 0 || kc > 0 || k > 0) ? 1u : 0u);
            tc_commit(o_bar);
        }
    }
    mbar_wait(o_bar, o_phase);  // last P.V done
    __syncwarp();
    tc_fence_after();

    // Epilogue: O row -> out[(seq, i)][(kvh*G + g)*HD + d].
    uint16_t* orow = out + (row0 + i) * static_cast<int64_t>(Hq) * HD + static_cast<int64_t>(kvh * G + g) * HD;
    for (int c0 = half * (HD / kPfParts); c0 < (half + 1) * (HD / kPfParts); c0 += 32) {
        float v[32];
        tmem_ld32(tO + lane_off + c0, v);  // warp-collective: every lane, stores predicated
        if (i < L) {
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8)
                *reinterpret_cast<uint4*>(orow + c0 + q8 * 8) =
                    make_uint4(pack2(v[q8 * 8], v[q8 * 8 + 1]), pack2(v[q8 * 8 + 2], v[q8 * 8 + 3]),
                               pack2(v[q8 * 8 + 4], v[q8 * 8 + 5]), pack2(v[q8 * 8 + 6], v[q8 * 8 + 7]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
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

namespace kl {
int g_prefill_tc = 2;  // kl_tune(KL_TUNE_PREFILL_TC, ...): 2 = 64-key blocks (default), 1 = 128-key blocks, 0 = CUDA cores
int g_decode_mma = 1;  // kl_tune(KL_TUNE_DECODE_MMA, ...)
int g_decode_hg = 0;   // kl_tune(KL_TUNE_DECODE_HG, ...): KV heads per decode work item (0 = auto)
int g_decode_stages = 0;  // kl_tune(KL_TUNE_DECODE_STAGES, ...): ring depth of the tensor-core decode kernel (0 = 3)
int g_attn_kv_evict_first = 1;  // kl_tune(KL_TUNE_ATTN_KV_EVICT_FIRST, ...): K/V read once per step
int g_rope_tok = 1;    // kl_tune(KL_TUNE_ROPE_TOKEN_BLOCKS, ...)

static int attn_sm_count() {
    static const int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            return v;
        cudaGetLastError();
        return 148;
    }();
    return n;
}
}

extern "C" int kl_rope_kv_append(uint16_t* qkv, int64_t T, int Hq, int Hkv, int hd, const int32_t* pos,
                                 const int32_t* seq, float rope_theta, uint16_t* k_cache, uint16_t* v_cache, int cap,
                                 int sink, int chunk_last_pos, cudaStream_t stream) {
    if (T < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || hd % 2 || cap <= sink || sink < 0) return KL_EINVAL;
    if (!qkv || !pos || !seq || !k_cache || !v_cache) return KL_EINVAL;
    if (T == 0) return KL_OK;
    // Block per token for prefill-sized calls; decode-sized calls (a few
    // dozen tokens) spread better with a thread per element.
    if (g_rope_tok && T >= 4 * 148 && hd % 8 == 0 && T <= 0x7fffffff &&
        ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(k_cache) | reinterpret_cast<uintptr_t>(v_cache)) & 15) == 0) {
        if (int rc_ = launch_pdl(rope_append_tok_kernel, dim3(static_cast<unsigned>(T)), dim3(kRopeThreads), static_cast<size_t>(hd) * 4, stream, qkv, Hq, Hkv, hd, pos, seq, rope_theta, k_cache, v_cache, cap, sink, chunk_last_pos)) return rc_;
        return check_launch();
    }
    const int64_t n = T * ((static_cast<int64_t>(Hq) + 2 * Hkv) * (hd / 2));
    if (int rc_ = launch_pdl(rope_append_kernel, dim3(static_cast<int>((n + 255) / 256)), dim3(256), 0, stream, qkv, T, Hq, Hkv, hd, pos, seq,
                                                                               rope_theta, k_cache, v_cache, cap, sink,
                                                                               chunk_last_pos)) return rc_;
    return check_launch();
}

extern "C" int kl_rope_kv_append_deferred(const float* qkv_part, int splits, int64_t part_rows, uint16_t* qkv,
                                          int64_t T, int Hq, int Hkv, int hd, const int32_t* pos, const int32_t* seq,
                                          float rope_theta, uint16_t* k_cache, uint16_t* v_cache, int cap, int sink,
                                          int chunk_last_pos, cudaStream_t stream) {
    if (T < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || hd % 2 || cap <= sink || sink < 0 || splits < 1 || splits > 4 ||
        T > part_rows)
        return KL_EINVAL;
    if (!qkv_part || !qkv || !pos || !seq || !k_cache || !v_cache) return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int64_t se = part_rows * (static_cast<int64_t>(Hq) + 2 * Hkv) * hd;
    if (hd % 8 == 0 && (reinterpret_cast<uintptr_t>(qkv_part) & 15) == 0 && (reinterpret_cast<uintptr_t>(qkv) & 7) == 0 &&
        ((reinterpret_cast<uintptr_t>(k_cache) | reinterpret_cast<uintptr_t>(v_cache)) & 7) == 0) {
        const int64_t nv = T * ((static_cast<int64_t>(Hq) + 2 * Hkv) * (hd / 8));
        return launch_pdl(rope_append_deferred_vec_kernel, dim3(static_cast<unsigned>((nv + 255) / 256)), dim3(256),
                          0, stream, qkv_part, splits, se, qkv, T, Hq, Hkv, hd, pos, seq, rope_theta, k_cache, v_cache,
                          cap, sink, chunk_last_pos);
    }
    const int64_t n = T * ((static_cast<int64_t>(Hq) + 2 * Hkv) * (hd / 2));
    return launch_pdl(rope_append_deferred_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, stream,
                      qkv_part, splits, se, qkv, T, Hq, Hkv, hd, pos, seq, rope_theta, k_cache, v_cache, cap, sink,
                      chunk_last_pos);
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

extern "C" int64_t kl_attn_decode_workspace_bytes(int64_t T, int Hq, int hd, int cap) {
    if (T <= 0 || Hq <= 0 || hd <= 0 || cap <= 0) return 0;
    const int64_t chunks = (cap + kDecChunk - 1) / kDecChunk;
    // fp32 partials (max, sum, o) per (token, chunk, q head) + one 64-bit
    // segment counter per (token, KV head group).
    return T * chunks * Hq * (static_cast<int64_t>(hd) + 2) * 4 + T * Hq * 8 + 64;
}

// 3D view of a KV cache [rows = cache_seqs * cap][Hkv * hd] for the decode
// kernel: dims (64 columns, rows, 64-column chunks), box (64, 16 slots, the
// group's chunks), 128B swizzle with the slot as the swizzle row.
static int make_kv_map(CUtensorMap* map, const void* base, int64_t rows, int row_elems, int chunks_per_box) {
    const MapKey key{base, rows, row_elems, -kDmSlots, -chunks_per_box};  // negative: this layout's own key space
    if (map_cache_get(key, map)) return 0;
    EncodeFn enc = encoder();
    if (enc == nullptr) return KL_ENODEV;
    const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(row_elems / 64)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_elems) * 2, 128};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kDmSlots), static_cast<cuuint32_t>(chunks_per_box)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return KL_EINVAL;
    map_cache_put(key, map);
    return 0;
}

extern "C" int kl_attn_decode_ws2(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq,
                                  int64_t T, int Hq, int Hkv, int hd, const uint16_t* k_cache, const uint16_t* v_cache,
                                  int64_t cache_seqs, int cap, int sink, float scale, uint16_t* out, void* workspace,
                                  int64_t workspace_bytes, cudaStream_t stream) {
    if (hd != 128 && hd != 64) return KL_EUNSUPPORTED;
    if (T < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || cap <= sink || cache_seqs < 0 || !q || !pos || !seq || !out)
        return KL_EINVAL;
    if (T == 0) return KL_OK;
    const int G = Hq / Hkv;
    if (G > 8) return KL_EUNSUPPORTED;
    const int64_t need = kl_attn_decode_workspace_bytes(T, Hq, hd, cap);
    const size_t smem = static_cast<size_t>(kDecChunk) * (Hkv * hd + kKPad) * 2 +
                        static_cast<size_t>(kDecChunk) * Hkv * hd * 2 + static_cast<size_t>(Hq) * hd * 4 +
                        static_cast<size_t>(Hq) * kDecChunk * 4 + 16;
    if (workspace == nullptr || workspace_bytes < need || smem > 200 * 1024 || q_stride % 8 != 0 ||
        (reinterpret_cast<uintptr_t>(k_cache) & 15) || (reinterpret_cast<uintptr_t>(v_cache) & 15))
        return kl_attn_decode(q, q_stride, pos, seq, T, Hq, Hkv, hd, k_cache, v_cache, cap, sink, scale, out, stream);
    const int n_chunks = (cap + kDecChunk - 1) / kDecChunk;
    float* part_ml = static_cast<float*>(workspace);
    float* part_o = part_ml + T * n_chunks * Hq * 2;
    // KV heads per CTA work item. With enough (token, head-group) pairs to
    // fill the GPU (>= 80 % of the SMs), each CTA takes whole pairs and no
    // token is split; otherwise the widest group and split tokens.
    int HG = std::min(Hkv, kDmMaxHG);
    int whole = 0;
    for (int hg_try = HG; hg_try >= 1; hg_try /= 2) {
        if (Hkv % hg_try) continue;
        if (g_decode_hg > 0 && hg_try != g_decode_hg) continue;  // forced group width (tuning)
        if (T * (Hkv / hg_try) * 5 >= static_cast<int64_t>(attn_sm_count()) * 4) {
            HG = hg_try;
            whole = 1;
            break;
        }
    }
    if (g_decode_hg > 0 && Hkv % g_decode_hg == 0 && g_decode_hg <= kDmMaxHG) HG = g_decode_hg;
    if (g_decode_mma && cache_seqs > 0 && Hkv % HG == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
        static_assert(kDmSlots == kDecChunk, "workspace layout shared with the per-chunk kernel");
        auto ring_bytes_n = [&](int hg, int stages) {
            const size_t stage = (static_cast<size_t>(2) * kDmSlots * hg * hd * 2 + static_cast<size_t>(hg) * G * hd * 2 +
                                  1023) & ~static_cast<size_t>(1023);
            return stages * stage + 1024 + 2 * stages * 8;
        };
        // Ring depth: 3 stages keep two CTAs per SM; when the whole (token,
        // group) pairs fit one CTA per SM anyway, a 4th stage is free smem and
        // streams faster (64 tokens x 2 groups: 21.0 -> 17.6 us).
        int nst = kDmStages;
        if (g_decode_stages > 0)
            nst = g_decode_stages;
        else if (whole && T * (Hkv / HG) <= attn_sm_count() && ring_bytes_n(HG, kDmStages + 1) <= 227 * 1024)
            nst = kDmStages + 1;
        auto ring_bytes = [&](int hg) { return ring_bytes_n(hg, nst); };
        // Wide GQA groups (e.g. 48 q / 8 kv heads with split tokens) can
        // overflow shared memory with all KV heads in one item: narrow the
        // item (HG stays a divisor of Hkv) until the ring fits.
        while (ring_bytes(HG) > 227 * 1024 && HG > 1 && Hkv % (HG / 2) == 0) HG /= 2;
        CUtensorMap mk, mv;
        const int64_t rows = cache_seqs * cap;
        int rc = make_kv_map(&mk, k_cache, rows, Hkv * hd, HG * hd / 64);
        if (rc) return rc;
        rc = make_kv_map(&mv, v_cache, rows, Hkv * hd, HG * hd / 64);
        if (rc) return rc;
        const size_t msmem = ring_bytes(HG);
        if (msmem > 227 * 1024) return KL_EUNSUPPORTED;
        // (A deeper ring at one CTA per SM measured the same as two CTAs with
        // three stages each.)
        auto kern = hd == 128 ? attn_decode_mma_kernel<128> : attn_decode_mma_kernel<64>;
        KL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem)));
        // Occupancy per (hd, HG, smem), queried once; several host threads
        // (loopback expert-parallel engines) may launch concurrently.
        static int occ_cache[2][kDmMaxHG + 1] = {};
        static size_t occ_smem[2][kDmMaxHG + 1] = {};
        static std::mutex occ_mu;
        const int hi = hd == 128;
        int occ_now = 0;
        {
            std::lock_guard<std::mutex> lk(occ_mu);
            if (occ_smem[hi][HG] != msmem) {
                int occ = 0;
                KL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (HG + 1) * 32, msmem));
                occ_cache[hi][HG] = std::max(occ, 1);
                occ_smem[hi][HG] = msmem;
            }
            occ_now = occ_cache[hi][HG];
        }
        const int64_t n_items = T * (Hkv / HG) * n_chunks;
        const int ctas = static_cast<int>(std::min<int64_t>(whole ? n_items / n_chunks : n_items,
                                                            static_cast<int64_t>(attn_sm_count()) * occ_now));
        // Segment counters after the partials (8-byte aligned); tags are
        // quiet-NaN bit patterns, distinct per call.
        static std::atomic<uint32_t> epoch{1};
        const uint32_t tag = 0x7FC00000u | (epoch.fetch_add(1) & 0x3FFFFFu);
        auto* counters = reinterpret_cast<unsigned long long*>(
            (reinterpret_cast<uintptr_t>(part_o + T * n_chunks * Hq * hd) + 7) & ~uintptr_t(7));
        return launch_pdl(kern, dim3(ctas), dim3((HG + 1) * 32), msmem, stream, mk, mv, q, q_stride, pos, seq, Hq,
                          Hkv, HG, cap, scale * 1.4426950408889634f, part_o, part_ml, n_chunks, n_items, out, counters,
                          tag, whole, nst, g_decode_mma | (g_attn_kv_evict_first ? 4 : 0));
    }
    auto kern = hd == 128 ? attn_decode_split_kernel<128> : attn_decode_split_kernel<64>;
    KL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<dim3(static_cast<unsigned>(T), n_chunks), kDecThreads, smem, stream>>>(
        q, q_stride, pos, seq, Hq, Hkv, k_cache, v_cache, cap, scale, part_o, part_ml, n_chunks);
    KL_CUDA_TRY(cudaGetLastError());
    auto merge = hd == 128 ? attn_merge_kernel<128> : attn_merge_kernel<64>;
    merge<<<dim3(static_cast<unsigned>(T), Hq), hd, 0, stream>>>(part_o, part_ml, Hq, n_chunks, out);
    return check_launch();
}

extern "C" int kl_attn_decode_ws(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq,
                                 int64_t T, int Hq, int Hkv, int hd, const uint16_t* k_cache, const uint16_t* v_cache,
                                 int cap, int sink, float scale, uint16_t* out, void* workspace,
                                 int64_t workspace_bytes, cudaStream_t stream) {
    // Cache extent unknown: the per-chunk kernel (it never reads past a
    // sequence's retained slots).
    return kl_attn_decode_ws2(q, q_stride, pos, seq, T, Hq, Hkv, hd, k_cache, v_cache, 0, cap, sink, scale, out,
                              workspace, workspace_bytes, stream);
}

extern "C" int kl_attn_prefill(const uint16_t* qkv, int n_seq, int L, int Hq, int Hkv, int hd, int cap, int sink,
                               float scale, uint16_t* out, cudaStream_t stream) {
    if (hd != 128 && hd != 64) return KL_EUNSUPPORTED;
    if (n_seq < 0 || L < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || cap <= sink || !qkv || !out) return KL_EINVAL;
    const int64_t warps = static_cast<int64_t>(n_seq) * L * Hq;
    if (warps == 0) return KL_OK;
    const int G = Hq / Hkv;
    const int width = (Hq + 2 * Hkv) * hd;
    if (g_prefill_tc && 128 % G == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 && width % 8 == 0) {
        CUtensorMap mq, mkv;
        int rc = make_map(&mq, qkv, static_cast<int64_t>(n_seq) * L, width, 128 / G);
        if (rc) return rc;
        // g_prefill_tc 2: 64-key blocks with one V buffer (two CTAs per SM).
        const int keys = g_prefill_tc == 2 ? 64 : kPfKeys;
        rc = make_map(&mkv, qkv, static_cast<int64_t>(n_seq) * L, width, keys);
        if (rc) return rc;
        const int nch = hd / 64;
        const int vbuf = keys == 64 ? 1 : 2;
        const int smem = nch * 128 * 128 + (2 + vbuf) * nch * keys * 128 + (keys / 64) * 128 * 128 + 1024 + 128 +
                         4096;  // Q, 2 K, V, P, alignment, barriers, stats
        auto kern = keys == 64 ? (hd == 128 ? attn_prefill_tc_kernel<128, 64> : attn_prefill_tc_kernel<64, 64>)
                               : (hd == 128 ? attn_prefill_tc_kernel<128, 128> : attn_prefill_tc_kernel<64, 128>);
        KL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const dim3 grid((L + 128 / G - 1) / (128 / G), Hkv, n_seq);
        kern<<<grid, kPfThreads, smem, stream>>>(mq, mkv, L, Hq, Hkv, sink, cap - sink, scale, out);
        return check_launch();
    }
    auto kern = hd == 128 ? attn_prefill_kernel<128> : attn_prefill_kernel<64>;
    kern<<<static_cast<int>((warps + 7) / 8), 256, 0, stream>>>(qkv, n_seq, L, Hq, Hkv, cap, sink, scale, out);
    return check_launch();
}
