// SPDX-License-Identifier: Apache-2.0
// Host-side TMA descriptor encoding shared by the tcgen05 kernels: the
// driver's cuTensorMapEncodeTiled through the runtime entry-point query (no
// libcuda link dependency).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "common.cuh"

namespace kl {

constexpr int kTmaBoxK = 64;  // 64 bf16 = 128 bytes = one 128B-swizzle span

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn encoder() {
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

// Encoded descriptors are cached by (kind, address, shape, box): a map only
// encodes these, so a hit is always valid, and repeated launches over the
// same buffers (expert slots, activation scratch) skip the driver encode on
// the host's launch path.
struct MapKey {
    const void* base;
    int64_t rows, cols;
    int box_rows, kchunks;
    int layout = 0;  // 0 = row-major [rows][cols], 1 = K-blocked (see make_map_kblocked)
    bool operator==(const MapKey& o) const {
        return base == o.base && rows == o.rows && cols == o.cols && box_rows == o.box_rows && kchunks == o.kchunks &&
               layout == o.layout;
    }
};
// Direct-mapped, 1024 entries, guarded by a mutex (launch paths may run on
// several host threads).
inline bool map_cache_op(const MapKey& k, CUtensorMap* m, bool put) {
    struct Entry {
        MapKey key;
        CUtensorMap map;
        bool used;
    };
    static Entry table[1024];
    static std::mutex mu;
    const uint64_t h = (reinterpret_cast<uint64_t>(k.base) >> 8) * 0x9E3779B97F4A7C15ull ^
                       static_cast<uint64_t>(k.rows) * 0xC2B2AE3D27D4EB4Full ^ static_cast<uint64_t>(k.cols) * 31u ^
                       static_cast<uint64_t>(k.box_rows) * 131u ^ static_cast<uint64_t>(k.kchunks) * 7u ^
                       static_cast<uint64_t>(k.layout) * 0x51ED27u;
    Entry& e = table[(h >> 32) & 1023];
    std::lock_guard<std::mutex> lock(mu);
    if (put) {
        e.key = k;
        e.map = *m;
        e.used = true;
        return true;
    }
    if (!e.used || !(e.key == k)) return false;
    *m = e.map;
    return true;
}
inline bool map_cache_get(const MapKey& k, CUtensorMap* out) {
    return map_cache_op(k, out, false);
}
inline void map_cache_put(const MapKey& k, const CUtensorMap* m) { map_cache_op(k, const_cast<CUtensorMap*>(m), true); }

// Row-major bf16 matrix [rows, cols] viewed by TMA in boxes of [box_rows, 64].
inline int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    const MapKey key{base, rows, cols, box_rows, 0};
    if (map_cache_get(key, map)) return 0;
    EncodeFn enc = encoder();
    if (enc == nullptr) return KL_ENODEV;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTmaBoxK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return KL_EINVAL;
    map_cache_put(key, map);
    return 0;
}

// Row-major bf16 matrix [rows, cols] viewed as (64 columns, rows, cols / 64):
// one box = box_rows rows x kchunks consecutive 64-column chunks, landing as
// kchunks slabs of [box_rows][64] (each the same 128B-swizzled tile a 2D box
// gives), so a single copy covers several k-blocks.
inline int make_map_kchunks(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows, int kchunks) {
    const MapKey key{base, rows, cols, box_rows, kchunks};
    if (map_cache_get(key, map)) return 0;
    EncodeFn enc = encoder();
    if (enc == nullptr) return KL_ENODEV;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kTmaBoxK), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(cols / kTmaBoxK)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, static_cast<cuuint64_t>(kTmaBoxK) * 2};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(kTmaBoxK), static_cast<cuuint32_t>(box_rows),
                               static_cast<cuuint32_t>(kchunks)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return KL_EINVAL;
    map_cache_put(key, map);
    return 0;
}

// K-blocked bf16 weights ("KB" layout, kl_weights_kblock): the [rows, cols]
// matrix stored as cols/64 slabs, slab j = columns [64j, 64j+64) of every row,
// row-major inside the slab (128 bytes per row). Viewed as (64, rows, cols/64)
// with strides (128 B, rows*128 B), a box of box_rows x 64 x kchunks is
// kchunks contiguous runs of box_rows*128 bytes (16 KB for a 128-row weight
// tile) instead of box_rows strided 128-byte pieces, and lands in shared
// memory exactly like the row-major box (same 128B swizzle).
inline int make_map_kblocked(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows,
                             int kchunks) {
    MapKey key{base, rows, cols, box_rows, kchunks};
    key.layout = 1;
    if (map_cache_get(key, map)) return 0;
    EncodeFn enc = encoder();
    if (enc == nullptr) return KL_ENODEV;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kTmaBoxK), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(cols / kTmaBoxK)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kTmaBoxK) * 2, static_cast<cuuint64_t>(rows) * kTmaBoxK * 2};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(kTmaBoxK), static_cast<cuuint32_t>(box_rows),
                               static_cast<cuuint32_t>(kchunks)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return KL_EINVAL;
    map_cache_put(key, map);
    return 0;
}

}  // namespace kl
