/* SPDX-License-Identifier: Apache-2.0
 *
 * klotski/kernels.h — C-ABI of the hand-written sm_100a kernels behind the
 * Klotski layer-execution path. One entry point per compute op kind of the
 * reference schedule (proj/include/moesim/schedule.hpp:32-45), which the
 * reference only *prices* in its simulator (proj/src/simulator.cpp:13-17):
 *
 *   compute_gate      (schedule.cpp:340-353)  -> kl_gate_topk
 *   compute_expert    (schedule.cpp:355-372)  -> kl_permute + kl_expert_ffn + kl_combine
 *   compute_attention (schedule.cpp:313-338)  -> kl_rmsnorm, kl_gemm_bf16, kl_rope_kv_append
 *                                               (decode: kl_rmsnorm_rope_table + kl_gemm_bf16_qkv_rope),
 *                                                kl_attn_decode / kl_attn_prefill
 *   update_table / predict_hot (correlation.cpp:74-140, invoked from
 *   make_table_prefetcher, schedule.cpp:60-91) -> kl_coact_update, kl_predict_scores
 *
 * Conventions (all entry points):
 *   - plain device pointers and sizes; bf16 tensors are passed as uint16_t*;
 *   - caller-owned buffers, no hidden allocation, no host synchronisation;
 *   - enqueue-only on `stream`; not thread-safe per stream;
 *   - return 0 on success, a positive cudaError_t value on a CUDA failure,
 *     or a negative KL_E* code for invalid arguments (no exceptions cross
 *     the ABI; the C++ layer maps codes to moesim exceptions).
 *   - row-major layouts; "K-major" weights are [out_features, in_features].
 */
#ifndef KLOTSKI_KERNELS_H
#define KLOTSKI_KERNELS_H

#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KL_OK 0
#define KL_EINVAL (-1)      /* bad shape / pointer / alignment */
#define KL_EUNSUPPORTED (-2) /* shape outside what the kernel implements */
#define KL_ENODEV (-3)      /* no sm_100 device / driver entry point missing */

/* Version / capability probe. Returns the compiled ABI version. */
int kl_abi_version(void);
/* 1 if the current device is sm_100 and the kernels can launch, else 0. */
int kl_device_supported(void);
/* Human-readable message for a return code (static storage). */
const char* kl_error_string(int code);

/* ---- dense / grouped GEMM on tcgen05 (TMEM accumulators, TMA operands) ----
 * C[M,N] = A[M,K] * B[N,K]^T, bf16 in, fp32 accumulate.
 * epilogue: 0 = store bf16 C
 *           1 = store bf16 (C + R)          (R: bf16 [M,N], may alias C)
 *           2 = SwiGLU: B holds [W1; W3] stacked as two [N/2, K] halves at
 *               b and b + (N/2)*K; out[m, j] = silu(acc1) * acc3, C is [M, N/2]
 * Requirements: K % 64 == 0, N % 64 == 0 (N % 256 == 0 for epilogue 2),
 * lda == K, ldb == K (contiguous rows), 16-byte aligned pointers.
 * row_offset selects rows [row_offset, row_offset + M) of a taller A whose
 * total row count is a_rows (used for expert-major permuted activations).
 * workspace (may be NULL): fp32 scratch enabling deterministic K-splits for
 * small-M (weight-streaming) shapes; kl_gemm_workspace_bytes() is the size
 * the split heuristic would like (less -> fewer splits, never an error). */
int64_t kl_gemm_workspace_bytes(int M, int N, int K, int epilogue);
/* Decode shapes (M <= 256) with a workspace take the weight-streaming path:
 * activations as the MMA's N side (rows padded to 16), weights as its M side
 * read exactly once, one persistent CTA per SM over equal (tile, k-block)
 * ranges; split tiles are finished by the CTA holding their last k-block,
 * adding the fp32 partials of the others in ascending CTA order
 * (deterministic). Its workspace holds one partial slot per CTA plus a
 * flag page (a smaller workspace runs fewer CTAs). */
#define KL_TUNE_STREAM_GEMM 0 /* 1 = weight-streaming path for >= 40 MB of weights or M > 128 (default), 2 = always, 0 = off */
#define KL_TUNE_STREAM_NMMA 1 /* 128-row weight sub-tiles per activation tile: 1 (default) or 2 */
#define KL_TUNE_STREAM_STAGES 2 /* cap on the smem pipeline depth (2..16, default 8) */
#define KL_TUNE_STREAM_HINT 3   /* 1 = L2 evict_first (weights) / evict_last (activations) hints, 2 = weights evict_last too, 0 = none */
#define KL_TUNE_STREAM_CTAS_PER_SM 4 /* persistent CTAs per SM: 1 (default) or 2 */
#define KL_TUNE_PDL 5 /* 1 = decode-path kernels use programmatic dependent launch (default) */
#define KL_TUNE_PREFILL_TC 6 /* tcgen05 prefill attention: 2 = 64-key blocks, two CTAs per SM (default), 1 = 128-key blocks, 0 = CUDA-core fallback */
#define KL_TUNE_ROPE_TOKEN_BLOCKS 11 /* 1 = RoPE/KV append with a block per token and a shared cos/sin table (default), 0 = thread per element */
#define KL_TUNE_STREAM_KBLOCKS_PER_STAGE 12 /* weight-streaming GEMM: 64-column k-blocks per pipeline stage: 3 (default) = 2 where >= 2 stages fit, 2 = 2 where >= 3 stages fit (3D TMA boxes), 1 */
#define KL_TUNE_STREAM_EVEN_SPLIT 13 /* weight-streaming GEMM: grid of tiles x floor(SMs / tiles), each tile split into equal k-ranges (1) or, default, also near-equal ones (2: the last range takes the remainder); 0 = stream-K ranges over one CTA per SM */
#define KL_TUNE_STREAM_FUSED_FIXUP 16 /* weight-streaming GEMM: 1 (default) = owners add split partials during the epilogue pass (dedicated staging region), 0 = TMEM fixup first */
#define KL_TUNE_DECODE_STAGES 21 /* tensor-core decode attention: ring stages (0 = default 3) */
#define KL_TUNE_ATTN_KV_EVICT_FIRST 19 /* tensor-core decode attention: 1 (default) = K/V loads with an L2 evict-first policy, 0 = no hint */
#define KL_TUNE_DECODE_HG 18 /* tensor-core decode attention: KV heads per work item (0 = auto) */
#define KL_TUNE_DECODE_MMA 9 /* 1 = persistent mma.sync split-KV decode attention (default), 0 = per-chunk CUDA-core kernel */
#define KL_TUNE_GEMM_PERSISTENT 8 /* 1 = persistent double-buffered-TMEM kernel for compute-bound GEMMs (default) */
#define KL_TUNE_STREAM_WHOLE_TILES 7 /* pct: one whole weight tile per CTA when tiles >= pct% of the SMs (default 70, 0 = off) */
/* Process-wide tuning knobs for benchmarking (not thread-safe). */
int kl_tune(int knob, int value);
/* Benchmarking aids: per-CTA phase timestamps (ns, globaltimer) of the last
 * weight-streaming GEMM launched with the trace debug bit (12 per CTA; the
 * buffer is cleared after the read), and a 1-thread kernel that holds
 * `stream` until the host-mapped *flag becomes non-zero (launch-latency-free
 * timing of the work queued behind it). */
int kl_stream_trace(unsigned long long* host, int n_ctas);
int kl_debug_spin_flag(const int* flag, cudaStream_t stream);
/* Device timestamp: writes the GPU global timer (ns) into *dst (device
 * memory) when `stream` reaches this point; the engine's op-boundary marks. */
int kl_stamp(unsigned long long* dst, cudaStream_t stream);
/* The next launch by the calling host thread of a kernel that supports it
 * (weight-streaming GEMM, decode-sized row RMSNorm, block-per-token router)
 * writes the same mark into *dst itself -- from its first CTA once its stream
 * predecessor is done -- instead of a separate kl_stamp kernel (the op's first
 * kernel is then one launch earlier); the other launch paths of those entry
 * points issue kl_stamp(dst) before themselves. */
int kl_stamp_next_launch(unsigned long long* dst);
/* The op-END counterpart: the next launch by the calling host thread of a
 * kernel that supports it (the deferred-split GEMMs' streaming launch -- for
 * kl_expert_ffn_kb_deferred its down projection -- and the block-per-token
 * router) has its last CTA to finish write %globaltimer into *dst, counted on
 * *counter (device u32, zero before first use; the writer resets it).
 * kl_stamp_end_pending() clears a mark no launch took and returns 1 if there
 * was one (the caller then issues kl_stamp itself). */
int kl_stamp_end_next_launch(unsigned long long* dst, unsigned* counter);
int kl_stamp_end_pending(void);
int kl_gemm_bf16(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                 const uint16_t* b, int N, uint16_t* c, int ldc, const uint16_t* r,
                 int epilogue, void* workspace, int64_t workspace_bytes, cudaStream_t stream);

/* One expert's SwiGLU FFN over its contiguous rows of the permuted buffer:
 *   H = silu(X W1^T) * (X W3^T)   (bf16 [M, f] scratch)
 *   Y = H W2^T                     (bf16 rows [row_offset, row_offset+M) of y)
 * w13 = [W1 (f x d); W3 (f x d)], w2 = d x f, all bf16 and contiguous
 * (exactly moesim ModelSpec::expert_bytes = 3*d*f*2 bytes starting at w13
 * when w2 == w13 + 2*f*d). h_scratch must hold M*f bf16. workspace as for
 * kl_gemm_bf16 (shared by both GEMMs, used sequentially). */
int kl_expert_ffn(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d,
                  int f, const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch,
                  uint16_t* y, void* workspace, int64_t workspace_bytes, cudaStream_t stream);

/* K-blocked weights (the engine's expert storage format for bf16). A
 * row-major [rows, cols] bf16 matrix stored as cols/64 slabs, slab j holding
 * columns [64j, 64j+64) of every row, row-major inside the slab:
 *   kb[(j*rows + r)*64 + c] = w[r*cols + 64j + c]
 * Same bytes as row-major; a 128-row x 64-column weight tile is one
 * contiguous 16 KB run, so the weight stream reads HBM in long runs instead
 * of 128-byte pieces 2*cols bytes apart (tools/tma_pattern_probe.cu: 6.34 vs
 * 5.60 TB/s). Results are bit-identical to the row-major entry points.
 *   kl_weights_kblock: convert (src != dst, cols % 64 == 0, 16 B aligned).
 *   kl_gemm_bf16_kb / kl_expert_ffn_kb: as kl_gemm_bf16 / kl_expert_ffn with
 *   b (w13 = [W1; W3] as one [2f, d] matrix, w2 = [d, f]) K-blocked. */
int kl_weights_kblock(const uint16_t* src, int64_t rows, int64_t cols, uint16_t* dst, cudaStream_t stream);
int kl_gemm_bf16_kb(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                    const uint16_t* b, int N, uint16_t* c, int ldc, const uint16_t* r,
                    int epilogue, void* workspace, int64_t workspace_bytes, cudaStream_t stream);
int kl_expert_ffn_kb(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d,
                     int f, const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch,
                     uint16_t* y, void* workspace, int64_t workspace_bytes, cudaStream_t stream);

/* ---- 4-bit expert streaming ----
 * Q4T layout: the reference's HQQ format (quant.cpp:197-252: 4-bit codes,
 * groups of 64 along K, fp16 scale and zero, w = scale * (code - zero))
 * with the groups of each 128-row x 64-column tile stored as one contiguous
 * 4608-byte chunk [128 x 32 B nibble codes | 128 fp16 scales | 128 fp16
 * zeros], chunks ordered (row tile, k-block). A permutation of the
 * reference's QuantizedTensor groups: same codes / scales / zeros.
 * rows % 128 == 0, K % 64 == 0. */
int64_t kl_q4_bytes(int64_t rows, int64_t K);
/* Min-max fit per group (moesim::fit_minmax, mirrored bit-exactly). */
int kl_quantize_q4(const uint16_t* w, int64_t rows, int64_t K, uint8_t* out, cudaStream_t stream);
/* out = bf16(scale * (code - zero)) (fp32 ops; equals the reference's
 * dequantize() rounded to bf16). */
int kl_dequantize_q4(const uint8_t* q, int64_t rows, int64_t K, uint16_t* w, cudaStream_t stream);
/* Weight-streaming GEMM with the dequantisation fused into the producer:
 * packed tiles bulk-copied to shared memory, expanded to 128B-swizzled bf16
 * by the (otherwise idle) epilogue warps, consumed by tcgen05.mma. Same
 * semantics / epilogues as kl_gemm_bf16 with B = dequantised weights;
 * M <= 256 (larger M: kl_dequantize_q4 + kl_gemm_bf16); workspace required. */
int64_t kl_gemm_q4_workspace_bytes(int M, int N, int K, int epilogue);
int kl_gemm_q4(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K, const uint8_t* bq,
               int N, uint16_t* c, int ldc, const uint16_t* r, int epilogue, void* workspace,
               int64_t workspace_bytes, cudaStream_t stream);
/* Expert FFN over Q4T weights: w13q = Q4T of [W1; W3] (2f x d), w2q = Q4T of W2 (d x f). */
int kl_expert_ffn_q4(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d,
                     int f, const uint8_t* w13q, const uint8_t* w2q, uint16_t* h_scratch,
                     uint16_t* y, void* workspace, int64_t workspace_bytes, cudaStream_t stream);

/* ---- routing ----
 * Fused RMSNorm + router + top-k for T tokens (one warp per token):
 *   x2[t]   = bf16(h[t] * rsqrt(mean(h[t]^2) + eps) * norm_w)      (stored)
 *   logit[t,e] = sum_i x2[t,i] * wg[e,i]   (fp32, fixed FMA + butterfly order,
 *                                           mirrored bit-exactly by the oracle)
 *   idx[t, 0..k-1]: top-k by logit, ties -> lower expert id
 *   weight: score_mode 0 = softmax over the k selected logits (Mixtral),
 *           score_mode 1 = softmax over all E logits, selected probs (DeepSeek)
 * Also accumulates hist[e] += count (int32, atomics) if hist != NULL and
 * records first_pos[e] = min token-major position (t*k+j) if first_pos != NULL
 * (initialise first_pos to INT32_MAX). logits (fp32 [T,E]) may be NULL.
 * Requirements: d % 256 == 0, E <= 64, k <= 8. */
int kl_gate_topk(const uint16_t* h, const uint16_t* norm_w, const uint16_t* wg, int T, int d,
                 int E, int k, float eps, int score_mode, uint16_t* x2, float* logits,
                 int32_t* idx, float* weight, int32_t* hist, int32_t* first_pos,
                 cudaStream_t stream);

/* Stable counting sort of the R = T*k routed rows into expert-major order:
 *   counts[e], offsets[e] (exclusive scan, offsets[E] = R),
 *   pos[r] = offsets[e_r] + #{r' < r : e_r' == e_r},   row_token[pos[r]] = r / k,
 *   xp[pos[r], :] = x2[r / k, :]   (vectorised 16-byte copies; xp may be NULL).
 * workspace: >= kl_permute_workspace_bytes(R, E) bytes. */
int64_t kl_permute_workspace_bytes(int64_t R, int E);
/* Kernels one kl_permute call launches for R = T*k routed rows (1 scan-only
 * for R = 0, 2 for a single 1024-row chunk, else 3). */
int kl_permute_launches(int64_t R);
int kl_permute(const int32_t* idx, int64_t T, int k, int E, const uint16_t* x2, int d,
               int32_t* counts, int32_t* offsets, int32_t* pos, int32_t* row_token,
               uint16_t* xp, void* workspace, cudaStream_t stream);

/* Weighted combine with residual:
 *   out[t] = bf16( float(resid[t]) + sum_{j<k} weight[t,j] * float(y[pos[t*k+j]]) )
 * accumulated in fp32 in j order (fmaf), mirrored bit-exactly by the oracle.
 * out may alias resid. */
int kl_combine(const uint16_t* y, const int32_t* pos, const float* weight,
               const uint16_t* resid, int64_t T, int k, int d, uint16_t* out,
               cudaStream_t stream);

/* Trace-replay routing: overwrite the router's choice with forced ids
 * (token-major [T,k]) and recompute weights as the softmax of the router's
 * own logits at those ids (score_mode 0), plus hist / first_pos as above. */
int kl_route_override(const int32_t* forced, const float* logits, int T, int E, int k,
                      int32_t* idx, float* weight, int32_t* hist, int32_t* first_pos,
                      cudaStream_t stream);

/* out[t] = table[ids[t]] (bf16 rows of width d). */
int kl_embed(const int32_t* ids, const uint16_t* table, int64_t T, int d, uint16_t* out,
             cudaStream_t stream);
/* out[t] = first index of max(logits[t, :V]) (greedy decoding). */
int kl_argmax_bf16(const uint16_t* logits, int64_t T, int V, int32_t* out, cudaStream_t stream);

/* ---- correlation-aware prefetcher statistics (exact integer atomics) ----
 * layer == 0: marginal[e] += 1 for every id in cur (prev ignored).
 * layer  > 0: table[(layer-1)][a][b] += 1 for every token and every
 *             (a in prev[t, :k], b in cur[t, :k]).  table: int64 [L-1][E][E]. */
int kl_coact_update(const int32_t* prev, const int32_t* cur, int64_t T, int k, int E, int layer,
                    int64_t* table, int64_t* marginal, cudaStream_t stream);
/* score[b] = sum_a hist[a] * table[(layer-1)][a][b]  (layer > 0), int64. */
int kl_predict_scores(const int32_t* hist, const int64_t* table, int E, int layer,
                      int64_t* score, cudaStream_t stream);

/* ---- attention block pieces ---- */
/* out[t] = bf16(x[t] * rsqrt(mean(x[t]^2) + eps) * w), d % 256 == 0. */
int kl_rmsnorm(const uint16_t* x, const uint16_t* w, int64_t T, int d, float eps,
               uint16_t* out, cudaStream_t stream);

/* kl_rmsnorm for decode-sized calls (T <= 592) that also writes each row's
 * RoPE (cos, sin) table for kl_gemm_bf16_qkv_rope: table[t][i] (float pairs,
 * i < hd/2) at position pos[t]. KL_EUNSUPPORTED for larger T. */
int kl_rmsnorm_rope_table(const uint16_t* x, const uint16_t* w, int64_t T, int d, float eps,
                          uint16_t* out, const int32_t* pos, float rope_theta, int hd, float* table,
                          cudaStream_t stream);

/* The QKV projection with kl_rope_kv_append fused into its epilogue:
 * c[0:M] = a[row_offset:+M] @ b^T (b = [Hq+2Hkv heads * hd, K] row-major),
 * q and k heads rotated with the table from kl_rmsnorm_rope_table, k and v
 * rows appended to the caches (same layout and retention rule as
 * kl_rope_kv_append). Results are bit-identical to kl_gemm_bf16 followed by
 * kl_rope_kv_append. Weight-streaming path only (hd 128, decode-sized M,
 * workspace of kl_gemm_workspace_bytes): KL_EUNSUPPORTED otherwise, and the
 * caller runs the two separate calls. */
int kl_gemm_bf16_qkv_rope(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                          const uint16_t* b, int Hq, int Hkv, int hd, uint16_t* c, int ldc,
                          const float* rope_table, const int32_t* pos, const int32_t* seq,
                          uint16_t* k_cache, uint16_t* v_cache, int cap, int sink, int chunk_last_pos,
                          void* workspace, int64_t workspace_bytes, cudaStream_t stream);

/* Deferred-reduction expert FFN for decode (weight-streaming path, K-blocked
 * weights): the down projection's tile-aligned k-splits each write their fp32
 * accumulator rows to y_part[split][row][d] (split stride part_rows * d) and
 * no CTA waits for another; kl_combine_deferred sums them in the owner's
 * order, so FFN + combine are bit-identical to kl_expert_ffn_kb + kl_combine.
 * `splits` must be kl_expert_ffn_deferred_splits(M, d, f) (0 = this shape
 * does not run as tile-aligned splits: use kl_expert_ffn_kb). */
int kl_expert_ffn_deferred_splits(int M, int d, int f);
/* Deferred split reduction for any decode-sized [N, K] weight-streaming GEMM
 * (e.g. the QKV projection): c_part[split][row][N] fp32 (split stride
 * part_rows * N); splits = kl_gemm_deferred_splits(M, N, K) (0 = not on the
 * tile-aligned split path). b_kblocked: weights in the K-blocked layout. */
int kl_gemm_deferred_splits(int M, int N, int K);
int kl_gemm_bf16_deferred(const uint16_t* a, int64_t a_rows, int64_t row_offset, int M, int K,
                          const uint16_t* b, int N, int b_kblocked, float* c_part, int64_t part_rows,
                          int splits, void* workspace, int64_t workspace_bytes, cudaStream_t stream);
/* kl_gate_topk (decode-sized T <= 592, block-per-token path) whose input row
 * is first completed from a deferred o-projection: h = bf16(Σ splits in the
 * owner's order + h), written back to h, then RMSNorm / router / top-k as
 * kl_gate_topk. Equal bit for bit to the streaming GEMM's residual epilogue
 * on the same splits followed by kl_gate_topk. KL_EUNSUPPORTED off that path. */
int kl_gate_topk_deferred(uint16_t* h, const float* h_part, int splits, int64_t part_rows,
                          const uint16_t* norm_w, const uint16_t* wg, int T, int d, int E, int k, float eps,
                          int score_mode, uint16_t* x2, float* logits, int32_t* idx, float* weight,
                          int32_t* hist, int32_t* first_pos, cudaStream_t stream);
/* kl_rope_kv_append over the fp32 split partials of a deferred QKV GEMM:
 * each element summed in the owner's order and rounded to bf16 (what the
 * GEMM would have stored), then RoPE / KV append as kl_rope_kv_append; the
 * full qkv rows are written. */
int kl_rope_kv_append_deferred(const float* qkv_part, int splits, int64_t part_rows, uint16_t* qkv, int64_t T,
                               int Hq, int Hkv, int hd, const int32_t* pos, const int32_t* seq,
                               float rope_theta, uint16_t* k_cache, uint16_t* v_cache, int cap, int sink,
                               int chunk_last_pos, cudaStream_t stream);
int kl_expert_ffn_kb_deferred(const uint16_t* xp, int64_t rows_total, int64_t row_offset, int M, int d, int f,
                              const uint16_t* w13, const uint16_t* w2, uint16_t* h_scratch, float* y_part,
                              int64_t part_rows, int splits, void* workspace, int64_t workspace_bytes,
                              cudaStream_t stream);
/* kl_combine over the fp32 split partials of kl_expert_ffn_kb_deferred
 * (1 <= splits <= 4, split stride split_rows * d). */
int kl_combine_deferred(const float* y_part, int splits, int64_t split_rows, const int32_t* pos,
                        const float* weight, const uint16_t* resid, int64_t T, int k, int d, uint16_t* out,
                        cudaStream_t stream);

/* Rotary embedding on q/k of a fused qkv row [Hq*hd | Hkv*hd | Hkv*hd] at the
 * token's absolute position, rope applied in place to q; roped k and v are
 * written to the KV cache slot of that position. Cache layout per layer:
 *   k_cache/v_cache: [n_seq][cap][Hkv][hd] bf16,
 *   slot(p) = p < sink ? p : sink + (p - sink) % (cap - sink).
 * pos[t] = absolute position, seq[t] = cache sequence index. For a prefill
 * chunk whose last position is chunk_last_pos, only positions still retained
 * after the chunk are written (p < sink or p > chunk_last_pos - (cap-sink)),
 * so ring slots are never written twice; pass -1 for decode. */
int kl_rope_kv_append(uint16_t* qkv, int64_t T, int Hq, int Hkv, int hd, const int32_t* pos,
                      const int32_t* seq, float rope_theta, uint16_t* k_cache,
                      uint16_t* v_cache, int cap, int sink, int chunk_last_pos,
                      cudaStream_t stream);

/* Decode attention (one query token per sequence), GQA, over the retained
 * slots of each sequence: min(pos+1, cap) slots (sink + sliding window).
 * q: [T][Hq*hd] (stride q_stride elements), out: [T][Hq*hd] bf16. hd in {64, 128}. */
int kl_attn_decode(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq,
                   int64_t T, int Hq, int Hkv, int hd, const uint16_t* k_cache,
                   const uint16_t* v_cache, int cap, int sink, float scale, uint16_t* out,
                   cudaStream_t stream);

/* Split-KV decode attention (same semantics as kl_attn_decode): one CTA per
 * (token, 16-slot chunk) stages the chunk's K and V rows with bulk async
 * copies, then a merge kernel folds the chunks in fixed order. workspace >=
 * kl_attn_decode_workspace_bytes(T, Hq, hd, cap) (fp32 partials); with a
 * smaller/NULL workspace it runs kl_attn_decode. */
int64_t kl_attn_decode_workspace_bytes(int64_t T, int Hq, int hd, int cap);
int kl_attn_decode_ws(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq,
                      int64_t T, int Hq, int Hkv, int hd, const uint16_t* k_cache,
                      const uint16_t* v_cache, int cap, int sink, float scale, uint16_t* out,
                      void* workspace, int64_t workspace_bytes, cudaStream_t stream);
/* Same, with the cache extent: k_cache / v_cache hold cache_seqs sequences of
 * cap slots (rows = cache_seqs * cap). With the extent known the persistent
 * tensor-core kernel runs (3D TMA boxes of 16 slots, mma.sync scores and
 * p.V, fixed-order segment merge); cache_seqs = 0 selects the per-chunk
 * CUDA-core kernel, which kl_attn_decode_ws always uses. */
int kl_attn_decode_ws2(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq, int64_t T, int Hq,
                       int Hkv, int hd, const uint16_t* k_cache, const uint16_t* v_cache, int64_t cache_seqs, int cap,
                       int sink, float scale, uint16_t* out, void* workspace, int64_t workspace_bytes,
                       cudaStream_t stream);

/* Prefill (chunk) attention: T = n_seq * L query rows laid out [seq][L]; keys
 * and values read from the same qkv rows (post-rope), causal with the same
 * sink + window retention mask as decode (window = cap - sink). hd in {64, 128}.
 * On tcgen05 when 128 % (Hq/Hkv) == 0: the GQA group's query heads share one
 * 128-row MMA tile; S = QK^T and O = PV accumulate in TMEM (two-pass softmax,
 * P staged as bf16 in shared memory). */
int kl_attn_prefill(const uint16_t* qkv, int n_seq, int L, int Hq, int Hkv, int hd, int cap,
                    int sink, float scale, uint16_t* out, cudaStream_t stream);

/* ---- expert-parallel helpers ----
 * out[i] = map[in[i]]  (relabel global expert ids, e.g. destination-major). */
int kl_map_ids(const int32_t* in, int64_t n, const int32_t* map, int32_t* out, cudaStream_t stream);
/* out[c] = sum_r in[r*cols + c]  (int32 histogram rows -> one histogram). */
int kl_sum_rows_i32(const int32_t* in, int rows, int cols, int32_t* out, cudaStream_t stream);
/* dst[i] += src[i]  (apply an all-reduced co-activation delta). */
int kl_add_i64(int64_t* dst, const int64_t* src, int64_t n, cudaStream_t stream);

/* Deterministic synthetic bf16 init on device: v[i] = N(0, std) from a
 * SplitMix64 stream keyed by (seed, i) (Box-Muller), for weights/inputs. */
int kl_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, float std_dev,
                        cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* KLOTSKI_KERNELS_H */
