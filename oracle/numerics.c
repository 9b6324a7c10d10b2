/* SPDX-License-Identifier: Apache-2.0
 *
 * CPU numeric oracle for the B200 Klotski layer path — TEST INFRASTRUCTURE.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library; the product path never does.
 *
 * The reference (proj/, a discrete-event simulator) contains NO model math:
 * compute ops carry only token counts (schedule.cpp:313-372) priced by
 * simulator.cpp:13-17. The numerics below restate the MoE block the paper
 * describes (attention + MoE layer + two norms, softmax
 * gate activating top-k, output = weighted sum of the selected experts) in
 * the Mixtral form (RMSNorm, GQA attention with RoPE, SwiGLU experts).
 *   => numerics: PARITY UNPINNED against the reference (no reference code
 *      computes them); pinned instead by construction + tests:
 *      - gate logits / top-k / weights: bit-exact order restatement of
 *        kl_gate_topk (lane-strided fmaf chunks + xor butterfly);
 *      - permute, combine, co-activation counts, prefetch scores: bit-exact;
 *      - FFN, attention, rope, rmsnorm: fp32 references, compared within the
 *        tolerances stated in tests/.
 * Routing *indices* in trace-replay mode and every schedule/prefetch/planner
 * decision are pinned against the reference itself (oracle/_ref).
 *
 * Compiled with -ffp-contract=off so only the explicit fmaf() calls fuse.
 */
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf2f(uint16_t v) {
    uint32_t u = (uint32_t)v << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static inline uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

void orc_f32_to_bf16(const float* in, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = f2bf(in[i]);
}
void orc_bf16_to_f32(const uint16_t* in, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = bf2f(in[i]);
}

/* Warp-order dot product of kl_gate_topk: 32 lane partials over chunks of 8
 * (lane l covers c = l*8 + 256*j), fmaf in element order, then xor butterfly. */
static float warp_order_dot(const uint16_t* x, const uint16_t* w, int d) {
    float lane_acc[32];
    for (int l = 0; l < 32; ++l) {
        float acc = 0.f;
        for (int c = l * 8; c < d; c += 256)
            for (int i = 0; i < 8; ++i) acc = fmaf(bf2f(x[c + i]), bf2f(w[c + i]), acc);
        lane_acc[l] = acc;
    }
    for (int o = 16; o > 0; o >>= 1) {
        float nxt[32];
        for (int l = 0; l < 32; ++l) nxt[l] = lane_acc[l] + lane_acc[l ^ o];
        memcpy(lane_acc, nxt, sizeof nxt);
    }
    return lane_acc[0];
}

/* Router from a given normalised input x2 (teacher forcing): logits, top-k
 * (ties -> lower id), weights (mode 0 Mixtral / mode 1 softmax-over-all). */
void orc_gate_topk(const uint16_t* x2, const uint16_t* wg, int T, int d, int E, int k, int score_mode,
                   float* logits, int32_t* idx, float* weight) {
#pragma omp parallel for schedule(static)
    for (int t = 0; t < T; ++t) {
        float lg[1024];
        for (int e = 0; e < E; ++e) lg[e] = warp_order_dot(x2 + (int64_t)t * d, wg + (int64_t)e * d, d);
        if (logits) memcpy(logits + (int64_t)t * E, lg, sizeof(float) * E);
        unsigned char taken[1024];
        memset(taken, 0, (size_t)E);
        int sel[64];
        float val[64];
        for (int j = 0; j < k; ++j) {
            int best = -1;
            float bv = 0.f;
            for (int e = 0; e < E; ++e) {
                if (taken[e]) continue;
                if (best < 0 || lg[e] > bv) {
                    best = e;
                    bv = lg[e];
                }
            }
            taken[best] = 1;
            sel[j] = best;
            val[j] = bv;
        }
        float p[64], s = 0.f;
        if (score_mode == 0) {
            for (int j = 0; j < k; ++j) s += (p[j] = expf(val[j] - val[0]));
        } else {
            float mx = lg[0];
            for (int e = 1; e < E; ++e) mx = fmaxf(mx, lg[e]);
            for (int e = 0; e < E; ++e) s += expf(lg[e] - mx);
            for (int j = 0; j < k; ++j) p[j] = expf(val[j] - mx);
        }
        for (int j = 0; j < k; ++j) {
            idx[(int64_t)t * k + j] = sel[j];
            weight[(int64_t)t * k + j] = p[j] / s;
        }
    }
}

void orc_rmsnorm(const uint16_t* x, const uint16_t* w, int64_t T, int d, float eps, uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        const uint16_t* r = x + t * d;
        double ss = 0.0;
        for (int i = 0; i < d; ++i) ss += (double)bf2f(r[i]) * bf2f(r[i]);
        const float rstd = (float)(1.0 / sqrt(ss / d + eps));
        for (int i = 0; i < d; ++i) out[t * d + i] = f2bf((bf2f(r[i]) * rstd) * bf2f(w[i]));
    }
}

/* Stable counting sort (the definition kl_permute must reproduce bit-exactly). */
void orc_permute(const int32_t* idx, int64_t T, int k, int E, int32_t* counts, int32_t* offsets, int32_t* pos,
                 int32_t* row_token) {
    const int64_t R = T * k;
    for (int e = 0; e < E; ++e) counts[e] = 0;
    for (int64_t r = 0; r < R; ++r) counts[idx[r]]++;
    int32_t acc = 0;
    for (int e = 0; e < E; ++e) {
        offsets[e] = acc;
        acc += counts[e];
    }
    offsets[E] = acc;
    int32_t* fill = (int32_t*)calloc((size_t)E, sizeof(int32_t));
    for (int64_t r = 0; r < R; ++r) {
        const int e = idx[r];
        const int32_t p = offsets[e] + fill[e]++;
        pos[r] = p;
        if (row_token) row_token[p] = (int32_t)(r / k);
    }
    free(fill);
}

void orc_combine(const uint16_t* y, const int32_t* pos, const float* weight, const uint16_t* resid, int64_t T, int k,
                 int d, uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t)
        for (int i = 0; i < d; ++i) {
            float acc = 0.f;
            for (int j = 0; j < k; ++j) acc = fmaf(weight[t * k + j], bf2f(y[(int64_t)pos[t * k + j] * d + i]), acc);
            out[t * d + i] = f2bf(bf2f(resid[t * d + i]) + acc);
        }
}

void orc_coact_update(const int32_t* prev, const int32_t* cur, int64_t T, int k, int E, int layer, int64_t* table,
                      int64_t* marginal) {
    for (int64_t t = 0; t < T; ++t) {
        if (layer == 0) {
            for (int j = 0; j < k; ++j) marginal[cur[t * k + j]]++;
        } else {
            int64_t* tab = table + (int64_t)(layer - 1) * E * E;
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) tab[prev[t * k + a] * E + cur[t * k + b]]++;
        }
    }
}

void orc_predict_scores(const int32_t* hist, const int64_t* table, int E, int layer, int64_t* score) {
    const int64_t* tab = table + (int64_t)(layer - 1) * E * E;
    for (int b = 0; b < E; ++b) {
        int64_t s = 0;
        for (int a = 0; a < E; ++a) s += (int64_t)hist[a] * tab[a * E + b];
        score[b] = s;
    }
}

/* C[M,N] = A[M,K] . B[N,K]^T in fp32 (bf16 inputs). Eight interleaved
 * partial sums per dot product (vectorisable without reassociation flags);
 * each thread converts one B row to fp32 and reuses it for every A row. */
void orc_gemm_f32(const uint16_t* a, const uint16_t* b, int64_t M, int64_t N, int64_t K, float* c) {
    float* af = (float*)malloc(sizeof(float) * M * K);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M * K; ++i) af[i] = bf2f(a[i]);
    const int64_t K8 = K & ~(int64_t)7;
#pragma omp parallel
    {
        float* brow = (float*)malloc(sizeof(float) * (K + 8));
#pragma omp for schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            for (int64_t i = 0; i < K; ++i) brow[i] = bf2f(b[n * K + i]);
            int64_t m = 0;
            for (; m + 4 <= M; m += 4) {  /* 4 A rows share each B load */
                const float* a0 = af + m * K;
                __m256 s0 = _mm256_setzero_ps(), s1 = s0, s2 = s0, s3 = s0;
                for (int64_t i = 0; i < K8; i += 8) {
                    const __m256 bv = _mm256_loadu_ps(brow + i);
                    s0 = _mm256_fmadd_ps(_mm256_loadu_ps(a0 + i), bv, s0);
                    s1 = _mm256_fmadd_ps(_mm256_loadu_ps(a0 + K + i), bv, s1);
                    s2 = _mm256_fmadd_ps(_mm256_loadu_ps(a0 + 2 * K + i), bv, s2);
                    s3 = _mm256_fmadd_ps(_mm256_loadu_ps(a0 + 3 * K + i), bv, s3);
                }
                float out[4][8];
                _mm256_storeu_ps(out[0], s0);
                _mm256_storeu_ps(out[1], s1);
                _mm256_storeu_ps(out[2], s2);
                _mm256_storeu_ps(out[3], s3);
                for (int r = 0; r < 4; ++r) {
                    float s = 0.f;
                    for (int j = 0; j < 8; ++j) s += out[r][j];
                    for (int64_t i = K8; i < K; ++i) s += a0[r * K + i] * brow[i];
                    c[(m + r) * N + n] = s;
                }
            }
            for (; m < M; ++m) {
                const float* ar = af + m * K;
                float s = 0.f;
                for (int64_t i = 0; i < K; ++i) s += ar[i] * brow[i];
                c[m * N + n] = s;
            }
        }
        free(brow);
    }
    free(af);
}

/* One expert: H = bf16(silu(X W1^T) * (X W3^T)), Y = bf16(H W2^T). */
void orc_expert_ffn(const uint16_t* x, int64_t M, int d, int f, const uint16_t* w13, const uint16_t* w2,
                    uint16_t* y) {
    float* g = (float*)malloc(sizeof(float) * M * 2 * (int64_t)f);
    orc_gemm_f32(x, w13, M, 2 * (int64_t)f, d, g);
    uint16_t* h = (uint16_t*)malloc(sizeof(uint16_t) * M * f);
    for (int64_t m = 0; m < M; ++m)
        for (int j = 0; j < f; ++j) {
            const float gv = g[m * 2 * f + j], uv = g[m * 2 * f + f + j];
            h[m * f + j] = f2bf(gv / (1.0f + expf(-gv)) * uv);
        }
    float* o = (float*)malloc(sizeof(float) * M * d);
    orc_gemm_f32(h, w2, M, d, f, o);
    orc_f32_to_bf16(o, M * d, y);
    free(g);
    free(h);
    free(o);
}

static int slot_of(int p, int cap, int sink) { return p < sink ? p : sink + (p - sink) % (cap - sink); }

void orc_rope_kv_append(uint16_t* qkv, int64_t T, int Hq, int Hkv, int hd, const int32_t* pos, const int32_t* seq,
                        float theta, uint16_t* kc, uint16_t* vc, int cap, int sink, int chunk_last_pos) {
    const int half = hd / 2;
    const int64_t width = (int64_t)(Hq + 2 * Hkv) * hd;
    for (int64_t t = 0; t < T; ++t) {
        uint16_t* row = qkv + t * width;
        const int p = pos[t];
        const int to_cache = chunk_last_pos < 0 || p < sink || p > chunk_last_pos - (cap - sink);
        const int64_t crow = ((int64_t)seq[t] * cap + slot_of(p, cap, sink)) * Hkv * hd;
        for (int head = 0; head < Hq + Hkv; ++head)
            for (int i = 0; i < half; ++i) {
                const float inv = powf(theta, -2.0f * (float)i / (float)hd);
                const float ang = (float)p * inv;
                const float cs = cosf(ang), sn = sinf(ang);
                uint16_t* base = row + (int64_t)head * hd;
                const float a = bf2f(base[i]), b = bf2f(base[i + half]);
                base[i] = f2bf(a * cs - b * sn);
                base[i + half] = f2bf(b * cs + a * sn);
                if (head >= Hq && to_cache) {
                    kc[crow + (int64_t)(head - Hq) * hd + i] = base[i];
                    kc[crow + (int64_t)(head - Hq) * hd + i + half] = base[i + half];
                }
            }
        if (to_cache)
            for (int h = 0; h < Hkv; ++h)
                memcpy(vc + crow + (int64_t)h * hd, row + (int64_t)(Hq + Hkv + h) * hd, sizeof(uint16_t) * hd);
    }
}

void orc_attn_decode(const uint16_t* q, int64_t q_stride, const int32_t* pos, const int32_t* seq, int64_t T, int Hq,
                     int Hkv, int hd, const uint16_t* kc, const uint16_t* vc, int cap, float scale, uint16_t* out) {
    const int G = Hq / Hkv;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        const int n = pos[t] + 1 < cap ? pos[t] + 1 : cap;
        float* s = (float*)malloc(sizeof(float) * n);
        for (int qh = 0; qh < Hq; ++qh) {
            const int kvh = qh / G;
            const uint16_t* qp = q + t * q_stride + (int64_t)qh * hd;
            const int64_t base = (int64_t)seq[t] * cap * Hkv * hd;
            float mx = -INFINITY;
            for (int j = 0; j < n; ++j) {
                const uint16_t* kp = kc + base + ((int64_t)j * Hkv + kvh) * hd;
                float acc = 0.f;
                for (int i = 0; i < hd; ++i) acc += bf2f(qp[i]) * scale * bf2f(kp[i]);
                s[j] = acc;
                if (acc > mx) mx = acc;
            }
            float sum = 0.f;
            for (int j = 0; j < n; ++j) sum += (s[j] = expf(s[j] - mx));
            for (int i = 0; i < hd; ++i) {
                float o = 0.f;
                for (int j = 0; j < n; ++j) o += s[j] * bf2f(vc[base + ((int64_t)j * Hkv + kvh) * hd + i]);
                out[t * Hq * hd + (int64_t)qh * hd + i] = f2bf(o / sum);
            }
        }
        free(s);
    }
}

void orc_attn_prefill(const uint16_t* qkv, int n_seq, int L, int Hq, int Hkv, int hd, int cap, int sink, float scale,
                      uint16_t* out) {
    const int G = Hq / Hkv, window = cap - sink;
    const int64_t width = (int64_t)(Hq + 2 * Hkv) * hd;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < (int64_t)n_seq * L; ++row) {
        const int sq = (int)(row / L), i = (int)(row % L);
        float* s = (float*)malloc(sizeof(float) * (i + 1));
        for (int qh = 0; qh < Hq; ++qh) {
            const int kvh = qh / G;
            const uint16_t* qp = qkv + row * width + (int64_t)qh * hd;
            float mx = -INFINITY;
            for (int j = 0; j <= i; ++j) {
                s[j] = -INFINITY;
                if (!(j < sink || j > i - window)) continue;
                const uint16_t* kp = qkv + ((int64_t)sq * L + j) * width + (int64_t)(Hq + kvh) * hd;
                float acc = 0.f;
                for (int x = 0; x < hd; ++x) acc += bf2f(qp[x]) * scale * bf2f(kp[x]);
                s[j] = acc;
                if (acc > mx) mx = acc;
            }
            float sum = 0.f;
            for (int j = 0; j <= i; ++j) sum += (s[j] = (s[j] == -INFINITY) ? 0.f : expf(s[j] - mx));
            for (int x = 0; x < hd; ++x) {
                float o = 0.f;
                for (int j = 0; j <= i; ++j)
                    if (s[j] != 0.f) o += s[j] * bf2f(qkv[((int64_t)sq * L + j) * width + (int64_t)(Hq + Hkv + kvh) * hd + x]);
                out[row * Hq * hd + (int64_t)qh * hd + x] = f2bf(o / sum);
            }
        }
        free(s);
    }
}

/* Same SplitMix64 Irwin-Hall(4) stream as kl_fill_normal_bf16 (bit-exact). */
static uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
void orc_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, float sd) {
    const float scale = 1.7320508075688772f * sd;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t z = splitmix(seed ^ ((uint64_t)i * 0xd1b54a32d192ed03ULL));
        const uint64_t w = splitmix(z);
        const float a = (float)(z & 0x3fffffu) + (float)((z >> 22) & 0x3fffffu);
        const float b = (float)(w & 0x3fffffu) + (float)((w >> 22) & 0x3fffffu);
        const float c = (a + b) * 0x1.0p-22f - 2.0f;
        dst[i] = f2bf(c * scale);
    }
}
