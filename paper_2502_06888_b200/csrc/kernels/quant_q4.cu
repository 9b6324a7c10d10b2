// SPDX-License-Identifier: Apache-2.0
// 4-bit expert weights for streaming: the reference's
// HQQ-style format (quant.cpp:197-252; QuantConfig bits 4, group 64, fp16
// scale and zero per group, w = scale * (code - zero)) with its groups laid
// out per 128-row x 64-column tile ("Q4T") so one tile of one expert matrix
// is one contiguous 4608-byte chunk: 128 x 32 bytes of little-endian nibble
// codes (element 2i in the low nibble of byte i, as the reference bit
// stream), 128 fp16 scales, 128 fp16 zeros. Relative to the reference's
// QuantizedTensor this is a permutation of whole groups, so codes, scales
// and zeros are bit-identical.
//
// kl_quantize_q4 fits each group with the reference's fit_minmax
// (quant.cpp: s = (hi - lo) / 15 in fp32, scale = fp16(s), zero = fp16(-lo/s),
// code = clamp(round(double(w) / scale + zero), 0, 15)), mirrored exactly
// (same IEEE operations), so codes match moesim::quantize's min-max fit.
#include <cuda_fp16.h>

#include "common.cuh"

namespace kl {
namespace {

constexpr int kQRows = 128, kQGroup = 64, kQChunk = kQRows * 32 + kQRows * 4;

__device__ __forceinline__ int64_t chunk_of(int64_t row, int64_t kb, int64_t KB) {
    return ((row / kQRows) * KB + kb) * kQChunk;
}

// One thread per group (row, k-block).
__global__ void quantize_q4_kernel(const uint16_t* __restrict__ w, int64_t rows, int64_t K, uint8_t* __restrict__ out) {
    const int64_t KB = K / kQGroup;
    const int64_t gidx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gidx >= rows * KB) return;
    const int64_t row = gidx / KB, kb = gidx % KB;
    const uint16_t* src = w + row * K + kb * kQGroup;
    float v[kQGroup];
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int i = 0; i < kQGroup; i += 8) {
        const uint4 q = *reinterpret_cast<const uint4*>(src + i);
        const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[i + 2 * k] = bf2f(static_cast<uint16_t>(ws[k] & 0xffffu));
            v[i + 2 * k + 1] = bf2f(static_cast<uint16_t>(ws[k] >> 16));
        }
    }
#pragma unroll
    for (int i = 0; i < kQGroup; ++i) {
        lo = fminf(lo, v[i]);
        hi = fmaxf(hi, v[i]);
    }
    __half hs, hz;
    if (lo == hi) {
        hs = __float2half_rn(1.0f);
        hz = __float2half_rn(-lo);
    } else {
        const float s = __fdiv_rn(__fsub_rn(hi, lo), 15.0f);
        hs = __float2half_rn(s);
        hz = __float2half_rn(__fdiv_rn(-lo, s));
    }
    const double sc = static_cast<double>(__half2float(hs)), zr = static_cast<double>(__half2float(hz));
    uint8_t* chunk = out + chunk_of(row, kb, KB);
    const int r = static_cast<int>(row % kQRows);
    uint32_t packed[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        uint32_t word = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const double qd = round(static_cast<double>(v[u * 8 + e]) / sc + zr);
            const int q = qd < 0.0 ? 0 : (qd > 15.0 ? 15 : static_cast<int>(qd));
            word |= static_cast<uint32_t>(q) << (4 * e);
        }
        packed[u] = word;
    }
    uint4* dst = reinterpret_cast<uint4*>(chunk + r * 32);
    dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    reinterpret_cast<uint16_t*>(chunk + kQRows * 32)[r] = __half_as_ushort(hs);
    reinterpret_cast<uint16_t*>(chunk + kQRows * 32 + kQRows * 2)[r] = __half_as_ushort(hz);
}

// bf16(scale * (code - zero)) with fp32 operations (the exact product of two
// floats rounded once, identical to the reference's double then float).
__global__ void dequantize_q4_kernel(const uint8_t* __restrict__ q, int64_t rows, int64_t K, uint16_t* __restrict__ w) {
    const int64_t KB = K / kQGroup;
    const int64_t gidx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gidx >= rows * KB) return;
    const int64_t row = gidx / KB, kb = gidx % KB;
    const uint8_t* chunk = q + chunk_of(row, kb, KB);
    const int r = static_cast<int>(row % kQRows);
    const float sc = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(chunk + kQRows * 32)[r]));
    const float zr = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(chunk + kQRows * 32 + kQRows * 2)[r]));
    const uint4 c0 = *reinterpret_cast<const uint4*>(chunk + r * 32);
    const uint4 c1 = *reinterpret_cast<const uint4*>(chunk + r * 32 + 16);
    const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    uint16_t* dst = w + row * K + kb * kQGroup;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float a = __fmul_rn(sc, __fsub_rn(static_cast<float>((cw[u] >> (8 * e)) & 15u), zr));
            const float b = __fmul_rn(sc, __fsub_rn(static_cast<float>((cw[u] >> (8 * e + 4)) & 15u), zr));
            pk[e] = pack2(a, b);
        }
        *reinterpret_cast<uint4*>(dst + u * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

}  // namespace
}  // namespace kl

extern "C" int64_t kl_q4_bytes(int64_t rows, int64_t K) {
    if (rows <= 0 || K <= 0 || rows % 128 || K % 64) return 0;
    return rows / 128 * (K / 64) * kl::kQChunk;
}

extern "C" int kl_quantize_q4(const uint16_t* w, int64_t rows, int64_t K, uint8_t* out, cudaStream_t stream) {
    if (!w || !out || rows <= 0 || K <= 0 || rows % 128 || K % 64) return KL_EINVAL;
    const int64_t groups = rows * (K / 64);
    kl::quantize_q4_kernel<<<static_cast<unsigned>((groups + 127) / 128), 128, 0, stream>>>(w, rows, K, out);
    return kl::check_launch();
}

extern "C" int kl_dequantize_q4(const uint8_t* q, int64_t rows, int64_t K, uint16_t* w, cudaStream_t stream) {
    if (!w || !q || rows <= 0 || K <= 0 || rows % 128 || K % 64) return KL_EINVAL;
    const int64_t groups = rows * (K / 64);
    kl::dequantize_q4_kernel<<<static_cast<unsigned>((groups + 127) / 128), 128, 0, stream>>>(q, rows, K, w);
    return kl::check_launch();
}
