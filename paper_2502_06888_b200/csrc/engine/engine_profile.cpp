// SPDX-License-Identifier: Apache-2.0
// Planner stage 1 on B200: "measure, then solve".
//
// The reference planner (make_plan / solve_min_n, planner.cpp:58-116 and
// 167-239) and cost model (build_cost_profile, cost.cpp:106-167) take a
// HardwareProfile of per-token compute rates and link bandwidths
// (model.hpp:43-58). Here those rates come from THIS engine's own kernels on
// the model's shapes, timed with CUDA events on one stream, plus the pinned
// host-to-device copy rate on one and on two concurrent copy streams:
//   attn_compute_per_token   = (rmsnorm + QKV GEMM + rope/KV append +
//                               attention + O GEMM with residual) / tokens
//                               of one batch (decode: bs tokens attending to
//                               the retained KV; prefill: bs x prompt_len)
//   gate_compute_per_token   = fused router (norm + gate + top-k) / tokens
//   expert_compute_per_token = expert FFN (SwiGLU GEMM + down GEMM) at the
//                              phase's mean routed rows per expert / rows
//   pcie_bandwidth           = pinned H2D bytes / time, 2 streams
// Scratch is cudaMalloc'd outside the engine arena and freed before it is
// allocated (the arena is exactly the HBM cap).
#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "klotski/kernels.h"

namespace klotski {

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw moesim::DeviceError(std::string("measure_profile: ") + what + ": " + cudaGetErrorString(e));
}
void kl_check(int rc, const char* what) {
    if (rc != 0) throw moesim::DeviceError(std::string("measure_profile: ") + what + ": " + kl_error_string(rc));
}

struct DevScratch {
    std::vector<void*> ptrs;
    ~DevScratch() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    T* get(int64_t elems) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(elems, 1)) * sizeof(T)), "cudaMalloc");
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

// Mean device time of `body` over `reps` runs after `warm` warm-up runs.
template <class F>
double time_ms(cudaStream_t st, int warm, int reps, F&& body) {
    for (int i = 0; i < warm; ++i) body();
    cudaEvent_t a, b;
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
    cuda_check(cudaEventRecord(a, st), "record");
    for (int i = 0; i < reps; ++i) body();
    cuda_check(cudaEventRecord(b, st), "record");
    cuda_check(cudaEventSynchronize(b), "sync");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / reps;
}

}  // namespace

std::string MeasuredProfile::to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "{\"phase\": \"" << phase << "\", \"tokens_per_batch\": " << tokens_per_batch
       << ", \"expert_rows\": " << expert_rows << ", \"kv_slots\": " << kv_slots << ", \"attn_ms\": " << attn_ms
       << ", \"gate_ms\": " << gate_ms << ", \"expert_ms\": " << expert_ms << ", \"attn_ps_per_token\": " << attn_ps
       << ", \"gate_ps_per_token\": " << gate_ps << ", \"expert_ps_per_token\": " << expert_ps
       << ", \"h2d_1stream_gbs\": " << h2d_1_gbs << ", \"h2d_2stream_gbs\": " << h2d_2_gbs
       << ", \"pcie_bandwidth\": " << pcie_bandwidth << "}";
    return os.str();
}

MeasuredProfile measure_profile(const EngineConfig& cfg, const std::string& phase) {
    const Dims& D = cfg.dims;
    const auto& w = cfg.workload;
    const bool prefill = phase == "prefill";
    if (!prefill && phase != "decode") throw moesim::ConfigError("measure_profile: phase must be decode or prefill");
    const int bs = w.batch_size;
    const int T = bs * (prefill ? w.prompt_len : 1);
    const int n = cfg.n_override ? *cfg.n_override : w.n_batches;
    // Retained KV slots per sequence at the middle of generation (decode) or
    // the prompt (prefill), as the engine's StreamingLLM / full policy keeps them.
    const int cap = std::max(2, cfg.retention.retained(w.prompt_len + w.gen_len));
    const int ctx = prefill ? w.prompt_len : std::min(cap, cfg.retention.retained(w.prompt_len + w.gen_len / 2));
    const int sink = cfg.retention.mode == moesim::KvRetentionPolicy::Mode::streaming ? std::min(cfg.retention.sink_tokens, cap - 1) : 0;
    // Mean routed rows per expert for one batch group of this phase.
    const int64_t routed = static_cast<int64_t>(n) * T * D.k;
    const int M = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(routed / D.E, 65536)));

    DevScratch mem;
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{st};
    const int qkvw = D.qkv_width();
    auto* wattn = mem.get<uint16_t>(D.attention_elems());
    auto* wgate = mem.get<uint16_t>(D.gate_elems());
    auto* wexp = mem.get<uint16_t>(D.expert_elems());
    auto* norm = mem.get<uint16_t>(D.d);
    auto* h = mem.get<uint16_t>(static_cast<int64_t>(T) * D.d);
    auto* x2 = mem.get<uint16_t>(static_cast<int64_t>(T) * D.d);
    auto* qkv = mem.get<uint16_t>(static_cast<int64_t>(T) * qkvw);
    auto* ao = mem.get<uint16_t>(static_cast<int64_t>(T) * D.Hq * D.hd);
    const int64_t kv_elems = static_cast<int64_t>(bs) * cap * D.Hkv * D.hd;
    auto* kc = mem.get<uint16_t>(kv_elems);
    auto* vc = mem.get<uint16_t>(kv_elems);
    auto* xp = mem.get<uint16_t>(static_cast<int64_t>(M) * D.d);
    auto* y = mem.get<uint16_t>(static_cast<int64_t>(M) * D.d);
    const int chunk = std::min(M, cfg.ffn_chunk_rows);
    auto* hs = mem.get<uint16_t>(static_cast<int64_t>(chunk) * D.f);
    auto* idx = mem.get<int32_t>(static_cast<int64_t>(T) * D.k);
    auto* wt = mem.get<float>(static_cast<int64_t>(T) * D.k);
    auto* pos = mem.get<int32_t>(T);
    auto* seq = mem.get<int32_t>(T);
    const int64_t ws_bytes = 40LL << 20;
    void* ws = mem.get<char>(ws_bytes);
    kl_check(kl_fill_normal_bf16(wattn, D.attention_elems(), 11, 0.02f, st), "init");
    kl_check(kl_fill_normal_bf16(wgate, D.gate_elems(), 12, 0.02f, st), "init");
    kl_check(kl_fill_normal_bf16(wexp, D.expert_elems(), 13, 0.02f, st), "init");
    kl_check(kl_fill_normal_bf16(h, static_cast<int64_t>(T) * D.d, 14, 1.0f, st), "init");
    kl_check(kl_fill_normal_bf16(xp, static_cast<int64_t>(M) * D.d, 15, 1.0f, st), "init");
    kl_check(kl_fill_normal_bf16(kc, kv_elems, 16, 1.0f, st), "init");
    kl_check(kl_fill_normal_bf16(vc, kv_elems, 17, 1.0f, st), "init");
    {
        std::vector<uint16_t> ones(D.d, 0x3f80);
        cuda_check(cudaMemcpy(norm, ones.data(), D.d * 2, cudaMemcpyHostToDevice), "norm");
        std::vector<int32_t> hp(T), hq(T);
        for (int t = 0; t < T; ++t) {
            hp[t] = prefill ? t % w.prompt_len : ctx - 1;
            hq[t] = prefill ? t / w.prompt_len : t;
        }
        cuda_check(cudaMemcpy(pos, hp.data(), T * 4, cudaMemcpyHostToDevice), "pos");
        cuda_check(cudaMemcpy(seq, hq.data(), T * 4, cudaMemcpyHostToDevice), "seq");
    }
    cuda_check(cudaStreamSynchronize(st), "init sync");

    const float scale = 1.0f / std::sqrt(static_cast<float>(D.hd));
    const uint16_t* wqkv = wattn;
    const uint16_t* wo = wattn + static_cast<int64_t>(qkvw) * D.d;
    MeasuredProfile out;
    out.phase = phase;
    out.tokens_per_batch = T;
    out.expert_rows = M;
    out.kv_slots = ctx;
    const int reps = prefill ? 3 : 20;
    out.attn_ms = time_ms(st, 2, reps, [&] {
        kl_check(kl_rmsnorm(h, norm, T, D.d, D.eps, x2, st), "rmsnorm");
        kl_check(kl_gemm_bf16(x2, T, 0, T, D.d, wqkv, qkvw, qkv, qkvw, nullptr, 0, ws, ws_bytes, st), "qkv");
        kl_check(kl_rope_kv_append(qkv, T, D.Hq, D.Hkv, D.hd, pos, seq, D.theta, kc, vc, cap, sink,
                                   prefill ? w.prompt_len - 1 : -1, st), "rope");
        if (prefill)
            kl_check(kl_attn_prefill(qkv, bs, w.prompt_len, D.Hq, D.Hkv, D.hd, cap, sink, scale, ao, st), "attn");
        else
            kl_check(kl_attn_decode_ws2(qkv, qkvw, pos, seq, T, D.Hq, D.Hkv, D.hd, kc, vc, bs, cap, sink, scale, ao, ws,
                                        ws_bytes, st), "attn");
        kl_check(kl_gemm_bf16(ao, T, 0, T, D.Hq * D.hd, wo, D.d, h, D.d, h, 1, ws, ws_bytes, st), "o proj");
    });
    out.gate_ms = time_ms(st, 2, reps, [&] {
        kl_check(kl_gate_topk(h, norm, wgate, T, D.d, D.E, D.k, D.eps, D.score_mode, x2, nullptr, idx, wt, nullptr,
                              nullptr, st), "gate");
    });
    out.expert_ms = time_ms(st, 2, prefill ? 3 : 20, [&] {
        for (int c = 0; c < M; c += chunk)
            kl_check((cfg.kblocked_experts && !cfg.quant ? kl_expert_ffn_kb : kl_expert_ffn)(
                         xp, M, c, std::min(chunk, M - c), D.d, D.f, wexp, wexp + 2LL * D.f * D.d, hs, y, ws, ws_bytes,
                         st), "expert ffn");
    });

    // Pinned H2D on one and on two concurrent copy streams.
    const size_t bytes = 256u << 20;
    void* host = nullptr;
    cuda_check(cudaHostAlloc(&host, bytes, cudaHostAllocDefault), "cudaHostAlloc");
    struct HostGuard {
        void* p;
        ~HostGuard() { cudaFreeHost(p); }
    } hguard{host};
    char* dst = mem.get<char>(static_cast<int64_t>(bytes));
    cudaStream_t st2;
    cuda_check(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking), "stream");
    StreamGuard guard2{st2};
    out.h2d_1_gbs = bytes / (time_ms(st, 1, 4, [&] {
                                 cuda_check(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, st), "h2d");
                             }) * 1e-3) / 1e9;
    cudaEvent_t fork, join;
    cuda_check(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&join, cudaEventDisableTiming), "event");
    out.h2d_2_gbs = bytes / (time_ms(st, 1, 4, [&] {
                                 const size_t half = bytes / 2;
                                 cuda_check(cudaEventRecord(fork, st), "fork");
                                 cuda_check(cudaStreamWaitEvent(st2, fork, 0), "fork wait");
                                 cuda_check(cudaMemcpyAsync(dst, host, half, cudaMemcpyHostToDevice, st), "h2d");
                                 cuda_check(cudaMemcpyAsync(dst + half, static_cast<char*>(host) + half, half,
                                                            cudaMemcpyHostToDevice, st2), "h2d");
                                 cuda_check(cudaEventRecord(join, st2), "join");
                                 cuda_check(cudaStreamWaitEvent(st, join, 0), "join wait");
                             }) * 1e-3) / 1e9;
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    cuda_check(cudaStreamSynchronize(st), "sync");

    auto ps = [](double ms, int64_t tokens) {
        return static_cast<moesim::duration_ps>(std::llround(ms * 1e9 / static_cast<double>(std::max<int64_t>(tokens, 1))));
    };
    out.attn_ps = std::max<moesim::duration_ps>(1, ps(out.attn_ms, T));
    out.gate_ps = std::max<moesim::duration_ps>(1, ps(out.gate_ms, T));
    out.expert_ps = std::max<moesim::duration_ps>(1, ps(out.expert_ms, M));
    out.pcie_bandwidth = std::max(out.h2d_1_gbs, out.h2d_2_gbs) * 1e9;
    return out;
}

}  // namespace klotski
