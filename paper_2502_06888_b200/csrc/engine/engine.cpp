// SPDX-License-Identifier: Apache-2.0
// B200 execution engine: setup (plan, arena, pinned host store, weights).
// See engine.hpp for the execution model. Reference anchors:
//   planning        make_plan / plan_placement (planner.cpp:167-239, placement.cpp:70-243)
//   warm-up table   prepare() (experiment.cpp:183-202)
//   op semantics    Builder::emit_* (schedule.cpp:155-372)
#include "engine.hpp"

#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <thread>

#include <nlohmann/json.hpp>

#include "klotski/kernels.h"
#include "splitmix.hpp"

namespace klotski {

using json = nlohmann::json;
using namespace moesim;

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw moesim::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

void kl_check(int rc, const char* what) {
    if (rc != 0) throw moesim::DeviceError(std::string(what) + ": " + kl_error_string(rc));
}

Dims preset_dims(const std::string& p) {
    Dims d;
    if (p == "mixtral-8x7b") {
        d = Dims{32, 4096, 14336, 32, 8, 128, 8, 2, 32000, 1e6f, 1e-5f, 0};
    } else if (p == "mixtral-8x22b") {
        d = Dims{56, 6144, 16384, 48, 8, 128, 8, 2, 32768, 1e6f, 1e-5f, 0};
    } else if (p == "deepseek-v2-lite") {
        // Fine-grained routed experts (64, top-6, softmax-over-all scores);
        // MLA is replaced by GQA attention of the same width.
        d = Dims{26, 2048, 1408, 16, 16, 128, 64, 6, 102400, 1e4f, 1e-6f, 1};
        d.n_shared = 2;
        d.f_shared = 1408;
    } else if (p == "tiny") {
        d = Dims{4, 512, 1792, 8, 2, 64, 8, 2, 1024, 1e6f, 1e-5f, 0};
    } else {
        throw ConfigError("unknown model preset '" + p + "'");
    }
    return d;
}

std::uint64_t tensor_seed(std::uint64_t base, int kind, int layer, int expert) {
    return mix64(base, (static_cast<std::uint64_t>(kind) << 48) ^ (static_cast<std::uint64_t>(layer) << 16) ^
                           static_cast<std::uint64_t>(expert + 1));
}

constexpr byte_count kGemmWorkspace = 40LL << 20;
constexpr int kKvSlots = 3;  // device KV slots when the KV tier is DRAM  // split-K partials for decode-shaped GEMMs
// Ops one step window can hold (op timestamps are sized by it): per layer n
// attentions, gates, KV loads and stores, up to 3 ops (load, compute,
// offload) per (expert, batch) for the per-batch variants, a few weight
// loads / offloads / window stages; slack for ops emitted ahead.
int64_t ops_per_step_bound(int layers, int64_t n, int64_t local_experts) {
    return static_cast<int64_t>(layers) * (4 * n + 3 * local_experts * n + 8) + 256;
}
constexpr int kKindExpert = 1, kKindAttn = 2, kKindGate = 3, kKindEmbed = 4, kKindHead = 5;

}  // namespace

EngineConfig parse_config(const std::string& text) {
    EngineConfig c;
    json j;
    try {
        j = text.empty() ? json::object() : json::parse(text);
    } catch (const json::exception& x) {
        throw ParseError(std::string("engine config: ") + x.what());
    }
    const json m = j.value("model", json::object());
    c.name = m.value("preset", "tiny");
    c.dims = preset_dims(c.name);
    Dims& D = c.dims;
    D.L = m.value("n_layers", D.L);
    D.d = m.value("d", D.d);
    D.f = m.value("f", D.f);
    D.Hq = m.value("heads", D.Hq);
    D.Hkv = m.value("kv_heads", D.Hkv);
    D.hd = m.value("head_dim", D.hd);
    D.E = m.value("experts", D.E);
    D.k = m.value("top_k", D.k);
    D.V = m.value("vocab", D.V);
    D.theta = m.value("rope_theta", D.theta);
    D.eps = m.value("norm_eps", D.eps);
    D.score_mode = m.value("score_mode", D.score_mode);
    D.n_shared = m.value("n_shared", D.n_shared);
    D.f_shared = m.value("f_shared", D.f_shared);
    if (D.n_shared < 0 || (D.n_shared > 0 && (D.fs() % 128 != 0 || D.f_shared <= 0)))
        throw ConfigError("engine: shared experts need n_shared * f_shared to be a multiple of 128");
    const json w = j.value("workload", json::object());
    c.workload.batch_size = w.value("batch_size", 4);
    c.workload.n_batches = w.value("n_batches", 4);
    c.workload.prompt_len = w.value("prompt_len", 8);
    c.workload.gen_len = w.value("gen_len", 4);
    if (w.contains("n_batches")) c.n_override = c.workload.n_batches;
    if (j.contains("n_override")) c.n_override = j["n_override"].get<int>();
    if (j.value("solve_n", false)) c.n_override.reset();
    c.plan_only = j.value("plan_only", false);
    c.hbm_cap = j.value("hbm_cap_bytes", c.hbm_cap);
    c.host_dram = j.value("host_dram_bytes", c.host_dram);
    c.pcie_bandwidth = j.value("pcie_bandwidth", c.pcie_bandwidth);
    c.attn_ps = j.value("attn_ps", c.attn_ps);
    c.gate_ps = j.value("gate_ps", c.gate_ps);
    c.expert_ps = j.value("expert_ps", c.expert_ps);
    if (j.contains("kv_retention")) {
        const json& r = j["kv_retention"];
        if (r.value("mode", "full") == "streaming") c.retention.mode = KvRetentionPolicy::Mode::streaming;
        c.retention.sink_tokens = r.value("sink_tokens", 4);
        c.retention.window_tokens = r.value("window_tokens", 256);
    }
    c.variant = variant_from_name(j.value("variant", "klotski"));
    c.replay = j.value("routing", "gate") == "replay";
    if (j.contains("skew")) {
        const json& s = j["skew"];
        const std::string kind = s.value("kind", "zipf");
        c.skew = kind == "uniform"  ? SkewSpec::uniform()
                 : kind == "markov" ? SkewSpec::markov(s.value("s", 1.5), s.value("p", 0.8))
                                    : SkewSpec::zipf(s.value("s", 1.5));
    }
    c.trace_seed = j.value("trace_seed", c.trace_seed);
    c.warmup_seed = j.value("warmup_seed", c.warmup_seed);
    c.weight_seed = j.value("weight_seed", c.weight_seed);
    c.host_distinct_layers = j.value("host_distinct_layers", 0);
    c.disk_dir = j.value("disk_dir", std::string());
    c.expert_slots = j.value("expert_slots", 0);
    c.ffn_chunk_rows = j.value("ffn_chunk_rows", 4096);
    {
        const std::string lay = j.value("expert_layout", std::string("kblocked"));
        if (lay != "kblocked" && lay != "row") throw ConfigError("engine: expert_layout must be 'kblocked' or 'row'");
        c.kblocked_experts = lay == "kblocked";
    }
    c.record_trace = j.value("record_trace", true);
    c.record_hidden = j.value("record_hidden", false);
    if (j.contains("ep")) {
        c.ep = true;
        c.ep_rank = j["ep"].value("rank", 0);
        c.ep_world = j["ep"].value("world", 1);
        c.ep_nccl_id = j["ep"].value("nccl_id", "");
        c.ep_backend = j["ep"].value("backend", "nccl");
        c.ep_group = j["ep"].value("group", "");
        if (c.ep_backend != "nccl" && c.ep_backend != "loopback")
            throw ConfigError("engine EP: backend must be 'nccl' or 'loopback'");
        if (c.ep_backend == "loopback" && c.ep_world > 1 && c.ep_group.empty())
            throw ConfigError("engine EP: the loopback backend needs a group name");
        if (c.ep_world < 1 || c.ep_rank < 0 || c.ep_rank >= c.ep_world || D.E % c.ep_world != 0)
            throw ConfigError("engine EP: need 0 <= rank < world and experts divisible by world");
        if (c.variant != Variant::klotski) throw ConfigError("engine EP: only the klotski variant is sharded");
        if (j.value("routing", "gate") != "gate") throw ConfigError("engine EP: routing must come from the gate");
    }
    c.prefill = j.value("prefill", true);
    if (j.contains("profile") && j["profile"].is_object() && j["profile"].contains("measure")) {
        c.measure_phase = j["profile"]["measure"].get<std::string>();
        if (c.measure_phase != "decode" && c.measure_phase != "prefill")
            throw ConfigError("engine: profile.measure must be 'decode' or 'prefill'");
    }
    if (j.contains("quant") && !j["quant"].is_null()) {
        moesim::QuantConfig q;
        q.bits = j["quant"].value("bits", 4);
        q.group_size = j["quant"].value("group_size", 64);
        if (q.bits != 4 || q.group_size != 64)
            throw ConfigError("engine: only 4-bit, group-64 expert streaming (Q4T) is executed");
        c.quant = q;
        if (c.ep) throw ConfigError("engine: quantised streaming is not combined with expert parallelism yet");
    }
    D.qkv_width();
    if (D.d % 256 || D.hd % 2 || D.Hq % D.Hkv || D.k > D.E || D.k > 8 || D.E > 64)
        throw ConfigError("engine: unsupported model dimensions");
    return c;
}

int ExpertSlotPool::acquire() {
    if (free_fifo.empty()) throw AccountingError("engine: expert slot pool exhausted");
    const int s = free_fifo.front();
    free_fifo.pop_front();
    return s;
}

void ExpertSlotPool::release_after(int slot, cudaEvent_t ev) {
    release[slot] = ev;
    has_release[slot] = ev != nullptr;
    free_fifo.push_back(slot);
}

Engine::Engine(const EngineConfig& cfg) : cfg_(cfg), D_(cfg.dims) {
    spec_.name = cfg_.name;
    spec_.n_layers = D_.L;
    spec_.n_experts_per_layer = D_.E;
    spec_.top_k = D_.k;
    spec_.expert_bytes = D_.expert_elems() * 2;
    spec_.attention_bytes = D_.attention_elems() * 2;
    spec_.gate_bytes = D_.gate_elems() * 2;
    spec_.kv_bytes_per_token = 2LL * D_.Hkv * D_.hd * 2;
    spec_.dtype = {"bf16", 16};
    spec_g_ = spec_;
    El_ = D_.E;
    if (cfg_.ep) {
        // The local shard is what this rank plans, places, streams and
        // schedules; the router and the correlation table stay global.
        ep_ = true;
        G_ = cfg_.ep_world;
        rank_ = cfg_.ep_rank;
        El_ = D_.E / G_;
        spec_.n_experts_per_layer = El_;
        spec_.top_k = std::min(D_.k, El_);
    }
    profile_.name = "b200";
    profile_.vram_capacity = cfg_.hbm_cap;
    profile_.dram_capacity = cfg_.host_dram;
    profile_.disk_capacity = 1'000'000'000'000LL;
    profile_.pcie_bandwidth = cfg_.pcie_bandwidth;
    profile_.disk_bandwidth = 3.0e9;
    profile_.attn_compute_per_token = cfg_.attn_ps;
    profile_.gate_compute_per_token = cfg_.gate_ps;
    profile_.expert_compute_per_token = cfg_.expert_ps;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (kl_device_supported() != 1) throw moesim::DeviceError("engine: device is not sm_100 (B200)");
    if (!cfg_.measure_phase.empty()) {
        // Paper stage 1: the planner's rates are measured on
        // this GPU with this engine's kernels before n and placement are solved.
        measured_ = measure_profile(cfg_, cfg_.measure_phase);
        profile_.attn_compute_per_token = measured_->attn_ps;
        profile_.gate_compute_per_token = measured_->gate_ps;
        profile_.expert_compute_per_token = measured_->expert_ps;
        profile_.pcie_bandwidth = measured_->pcie_bandwidth;
    }
    plan_memory();
    if (cfg_.plan_only) return;  // the planner's answer only: no HBM, host memory or streams
    allocate_device();
    allocate_host();
    for (auto& s : streams_) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&rb_stream_, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t* e : {&routing_ready_, &gates_done_, &scores_done_, &scores_ready_})
        cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreate(&step_begin_), "event");
    cuda_check(cudaEventCreate(&step_end_), "event");
    ep_init();
    init_weights();
    const detail::GroupShape shape{cfg_.workload.gen_len, D_.L, plan_.n_batches, cfg_.workload.batch_size,
                           cfg_.workload.prompt_len, spec_.top_k, El_};
    em_ = std::make_unique<detail::Emitter>(cfg_.variant, plan_, shape, ScheduleOptions{});
    // Trace containers: replayed routing and the routing actually executed.
    BatchGroupConfig g = cfg_.workload;
    g.n_batches = plan_.n_batches;
    if (cfg_.replay) replay_trace_ = generate_trace(spec_g_, g, cfg_.skew, cfg_.trace_seed);
    recorded_ = generate_trace(spec_g_, g, SkewSpec::uniform(), 0);
    recorded_.seed = 0;
    std::fill(recorded_.sel.begin(), recorded_.sel.end(), 0);
    host_marginal_ = table0_.marginal;
}

Engine::~Engine() {
    cudaDeviceSynchronize();
    ep_shutdown();
    for (auto& s : streams_)
        if (s) cudaStreamDestroy(s);
    for (auto& pool : event_pool_)
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (rb_stream_) cudaStreamDestroy(rb_stream_);
    for (cudaEvent_t e : {routing_ready_, gates_done_, scores_done_, scores_ready_})
        if (e) cudaEventDestroy(e);
    if (step_begin_) cudaEventDestroy(step_begin_);
    if (step_end_) cudaEventDestroy(step_end_);
    for (cudaEvent_t e : pool_.release) (void)e;
    if (arena_) cudaFree(arena_);
    for (void* p : host_blocks_) cudaFreeHost(p);
    if (disk_fd_ >= 0) ::close(disk_fd_);
}

void* Engine::take(byte_count bytes) {
    const byte_count aligned = (arena_used_ + 1023) & ~byte_count(1023);
    if (aligned + bytes > cfg_.hbm_cap)
        throw MemoryInfeasible("engine arena: " + std::to_string(aligned + bytes) + " B exceeds HBM cap " +
                                   std::to_string(cfg_.hbm_cap) + " B",
                               aligned + bytes - cfg_.hbm_cap, 0, 0);
    arena_used_ = aligned + bytes;
    return arena_ == nullptr ? nullptr : arena_ + aligned;
}

// The planner's working-set term is replaced by what this engine really
// keeps in HBM besides resident layers and KV: slot pools, scratch,
// embeddings/head, norms, routing buffers.
void Engine::plan_memory() {
    const BatchGroupConfig& w = cfg_.workload;
    // Warm-up trace -> correlation table + stats, as prepare() does.
    BatchGroupConfig warm = w;
    warm.n_batches = w.batch_size > 1 ? 2 : 4;
    const ActivationTrace wt =
        generate_trace(spec_g_, warm, cfg_.skew, cfg_.warmup_seed ? cfg_.warmup_seed : cfg_.trace_seed + 1);
    table0_ = build_table(wt, spec_g_);
    stats_ = compute_trace_stats(wt, D_.k);

    // Streamed tensors travel as Q4T when quantised (= the planner's
    // quantized_bytes, model_cost.cpp on_wire); resident ones stay bf16.
    expert_slot_bytes_ = cfg_.quant ? kl_q4_bytes(2LL * D_.f, D_.d) + kl_q4_bytes(D_.d, D_.f) : spec_.expert_bytes;
    attn_slot_bytes_ = cfg_.quant ? kl_q4_bytes(D_.qkv_width(), D_.d) + kl_q4_bytes(D_.d, static_cast<int64_t>(D_.Hq) * D_.hd)
                                  : spec_.attention_bytes;
    // The reference planner's own answer (its working-set formula,
    // placement.cpp:109-118): solved n and the KV-capped n.
    int n = 0;
    if (cfg_.n_override) {
        n = *cfg_.n_override;
    } else {
        const PipelinePlan ref = make_plan(spec_, profile_, w, stats_, cfg_.quant, ExpertLoadModel::measured, cfg_.retention);
        planner_solved_n_ = ref.solved_n_uncapped;
        planner_n_ = ref.n_batches;
        n = ref.n_batches;
    }
    // The engine's working set grows with n (the group's activations and
    // routed rows live in HBM), so a solved n is further capped to the
    // largest n whose real working set fits, the same monotone search the
    // reference uses for its KV cap (planner.cpp:195-229).
    if (plan_at(n)) return finish_plan();
    if (cfg_.n_override) {
        plan_at(n, /*rethrow=*/true);
        return;
    }
    if (!plan_at(1)) plan_at(1, /*rethrow=*/true);
    int lo = 1, hi = n - 1;
    while (lo < hi) {
        const int mid = lo + (hi - lo + 1) / 2;
        if (plan_at(mid))
            lo = mid;
        else
            hi = mid - 1;
    }
    plan_at(lo, true);
    memory_capped_n_ = lo;
    plan_.warnings.push_back("planner n=" + std::to_string(n) + " exceeds the engine's HBM working set; capped to n=" +
                             std::to_string(plan_.n_batches));
    finish_plan();
}

// One planning attempt at n with the engine's working set at n (and at the
// KV-capped n if the planner lowers it). false = MemoryInfeasible at n.
bool Engine::plan_at(int n, bool rethrow) {
    const BatchGroupConfig& w = cfg_.workload;
    const TraceStats stats = stats_;
    // KV offload (KV tier = DRAM): the cache of one (layer, batch) lives in a
    // device slot only between its load and its store; kKvSlots slots.
    bool kv_off = false;
    for (int attempt = 0; attempt < 4; ++attempt) {
        const int64_t seqs = static_cast<int64_t>(w.batch_size) * n;
        t_max_ = seqs * (cfg_.prefill ? w.prompt_len : 1);
        tb_max_ = static_cast<int64_t>(w.batch_size) * (cfg_.prefill ? w.prompt_len : 1);
        slots_ = cfg_.expert_slots > 0 ? cfg_.expert_slots : El_ + spec_.top_k;
        r_recv_max_ = ep_ ? static_cast<int64_t>(G_) * t_max_ * D_.k : 0;
        const int64_t Rx = std::max<int64_t>(t_max_ * D_.k, r_recv_max_);
        const int64_t R = t_max_ * D_.k;
        // One local expert can receive rows from every rank under EP, so the
        // FFN chunk is bounded by the exchange rows, not this rank's own.
        const int64_t chunk = std::min<int64_t>(cfg_.ffn_chunk_rows, std::max<int64_t>(Rx, 1));
        const int64_t chunk_own = std::min<int64_t>(cfg_.ffn_chunk_rows, std::max<int64_t>(R, 1));
        byte_count ws = 0;
        auto add = [&](byte_count b) { ws += ((b + 1023) / 1024) * 1024; };
        add(2 * attn_slot_bytes_);
        if (cfg_.quant) add(std::max(spec_.expert_bytes, spec_.attention_bytes));  // bf16 staging / dequant scratch
        add(2 * spec_.gate_bytes);
        for (int s = 0; s < slots_; ++s) add(expert_slot_bytes_);
        add(static_cast<byte_count>(D_.L) * 2 * D_.d * 2 + D_.d * 2);
        add(2LL * D_.V * D_.d * 2);
        add(2 * t_max_ * D_.d * 2);                                              // h, x2
        add(tb_max_ * (D_.d + D_.qkv_width() + D_.Hq * D_.hd) * 2);              // xa, qkv, ao
        add(5 * R * 4 + R * 4 + t_max_ * D_.E * 4);                              // idx x2, forced, pos, row_token, weight, logits
        add(2 * Rx * D_.d * 2);                                                   // xp, y
        add(chunk * D_.f * 2);                                                   // hs
        if (D_.fs() > 0) add(chunk_own * D_.fs() * 2);                           // shared-expert hidden
        add(kl_permute_workspace_bytes(Rx, D_.E));
        if (ep_) {  // exchange buffers, labels, counts, co-activation delta
            add(r_recv_max_ * D_.d * 2 * 2 + R * D_.d * 2);
            add((R + 3 * r_recv_max_) * 4 + (3LL * D_.E + 2 * El_ + 8) * 4);
            add((static_cast<int64_t>(D_.E) * D_.E + D_.E) * 8);
            if (cfg_.ep_backend == "loopback") add(static_cast<int64_t>(G_) * (D_.E * D_.E + D_.E) * 8);
        }
        // Split-K partials: the largest request of any small-M GEMM we issue.
        gemm_ws_bytes_ = 0;
        for (int64_t m : {int64_t{32}, int64_t{64}, int64_t{128}, int64_t{192}, int64_t{256}, tb_max_, seqs, Rx}) {
            // Largest GEMM row count this engine issues: own routed rows, a
            // batch, or (EP) the rows one local expert can receive.
            if (m > std::max({R, Rx, tb_max_})) continue;
            const int mi = static_cast<int>(m);
            gemm_ws_bytes_ = std::max({gemm_ws_bytes_, kl_gemm_workspace_bytes(mi, 2 * D_.f, D_.d, 2),
                                       kl_gemm_workspace_bytes(mi, D_.d, D_.f, 0),
                                       kl_gemm_workspace_bytes(mi, D_.qkv_width(), D_.d, 0),
                                       kl_gemm_workspace_bytes(mi, D_.d, D_.Hq * D_.hd, 1),
                                       kl_gemm_workspace_bytes(mi, D_.V, D_.d, 0)});
            if (D_.fs() > 0)
                gemm_ws_bytes_ = std::max({gemm_ws_bytes_, kl_gemm_workspace_bytes(mi, 2 * D_.fs(), D_.d, 2),
                                           kl_gemm_workspace_bytes(mi, D_.d, D_.fs(), 1)});
            if (cfg_.quant)
                gemm_ws_bytes_ = std::max({gemm_ws_bytes_, kl_gemm_q4_workspace_bytes(mi, 2 * D_.f, D_.d, 2),
                                           kl_gemm_q4_workspace_bytes(mi, D_.d, D_.f, 0),
                                           kl_gemm_q4_workspace_bytes(mi, D_.qkv_width(), D_.d, 0),
                                           kl_gemm_q4_workspace_bytes(mi, D_.d, D_.Hq * D_.hd, 1)});
        }
        // Decode attention partials (split-KV) share the same scratch.
        gemm_ws_bytes_ = std::max(gemm_ws_bytes_,
                                  kl_attn_decode_workspace_bytes(w.batch_size, D_.Hq, D_.hd,
                                                                 cfg_.retention.retained(w.prompt_len + w.gen_len)));
        // A smaller workspace only means fewer CTAs in the weight-streaming
        // GEMMs; keep it a small fraction of tight HBM caps.
        gemm_ws_bytes_ = std::min<int64_t>({gemm_ws_bytes_, kGemmWorkspace, std::max<int64_t>(256LL << 10, cfg_.hbm_cap / 256)});
        add(gemm_ws_bytes_);
        add(6 * t_max_ * 4 + 2 * (D_.E + 1) * 4);                                // pos/seq/seq_local/ids/next/last, counts/offsets
        add(seqs * D_.d * 2 + seqs * D_.V * 2);                                  // last_h, head logits
        add(2LL * n * D_.E * 4 + 2LL * D_.E * 8 + 64);                           // report
        add((static_cast<byte_count>(std::max(D_.L - 1, 0)) * D_.E * D_.E + D_.E) * 8);
        add(64 * 1024);
        add((2 * ops_per_step_bound(D_.L, n, El_) + 8) * 8);                     // op timestamps
        add(tb_max_ * D_.hd * 4);                                                // RoPE table
        if (defer_possible()) add(4LL * n * w.batch_size * D_.k * D_.d * 4);    // deferred FFN split partials
        if (defer_attn_possible())                                               // deferred QKV / o-proj partials
            add(4LL * w.batch_size * D_.qkv_width() * 4 + 4LL * n * w.batch_size * D_.d * 4);
        if (kv_off)
            add(static_cast<byte_count>(kKvSlots) * w.batch_size *
                cfg_.retention.retained(w.prompt_len + w.gen_len - 1) * spec_.kv_bytes_per_token);
        ws_bytes_ = ws;
        PlacementConfig pc;
        pc.working_set_override = ws;
        try {
            plan_ = make_plan(spec_, profile_, w, stats, cfg_.quant, ExpertLoadModel::measured, cfg_.retention, n, pc);
        } catch (const MemoryInfeasible&) {
            if (rethrow) throw;
            return false;
        }
        const bool off_now = plan_.placement.kv_tier == Tier::dram;
        if (plan_.n_batches == n && off_now == kv_off) break;
        n = plan_.n_batches;  // KV-capped: resize scratch for the capped n
        kv_off = off_now;     // KV slots join the working set
    }
    return true;
}

// Deferred split reduction applies to decode blocks of bf16 K-blocked experts
// on one GPU with one combine per block (not the per-batch simple variant).
bool Engine::defer_possible() const {
    return !cfg_.quant && !ep_ && cfg_.kblocked_experts && cfg_.variant != Variant::simple;
}
// The attention projections defer in every variant and under expert
// parallelism (each batch's router op follows its attention op); not with
// Q4T-streamed attention weights.
bool Engine::defer_attn_possible() const { return !cfg_.quant; }

void Engine::finish_plan() {
    kv_offload_ = plan_.placement.kv_tier == Tier::dram;
    if (kv_offload_ && ep_) throw ConfigError("engine: KV offload is not combined with expert parallelism yet");
    if (plan_.placement.any_disk() && ep_)
        throw ConfigError("engine: disk-tier placement is not combined with expert parallelism yet");
    kv_cap_ = plan_.placement.kv_retained_tokens;
    kv_sink_ = cfg_.retention.mode == KvRetentionPolicy::Mode::streaming ? std::min(cfg_.retention.sink_tokens, kv_cap_ - 1) : 0;
    kv_bytes_layer_ = kv_offload_ ? 0
                                  : static_cast<byte_count>(cfg_.workload.batch_size) * plan_.n_batches * kv_cap_ *
                                        spec_.kv_bytes_per_token;
    kv_slot_bytes_ = static_cast<byte_count>(cfg_.workload.batch_size) * kv_cap_ * spec_.kv_bytes_per_token;
}

void Engine::allocate_device() {
    // Dry run to size, then one arena of exactly the HBM cap.
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&arena_), static_cast<size_t>(cfg_.hbm_cap)), "cudaMalloc arena");
    arena_used_ = 0;
    const int n = plan_.n_batches;
    const int64_t seqs = static_cast<int64_t>(cfg_.workload.batch_size) * n;
    const int64_t R = t_max_ * D_.k;
    auto bf = [&](int64_t elems) { return static_cast<uint16_t*>(take(elems * 2)); };
    auto i32 = [&](int64_t elems) { return static_cast<int32_t*>(take(elems * 4)); };

    if (plan_.cost.expert_transfer_bytes != expert_slot_bytes_ || plan_.cost.attention_transfer_bytes != attn_slot_bytes_)
        throw AccountingError("engine: streamed tensor bytes disagree with the plan's transfer bytes");
    attn_slot_ = {bf(attn_slot_bytes_ / 2), bf(attn_slot_bytes_ / 2)};
    if (cfg_.quant) wscratch_ = bf(std::max(D_.expert_elems(), D_.attention_elems()));
    gate_slot_ = {bf(D_.gate_elems()), bf(D_.gate_elems())};
    attn_slot_busy_.assign(2, 0);
    gate_slot_busy_.assign(2, 0);
    attn_slot_release_.assign(2, nullptr);
    gate_slot_release_.assign(2, nullptr);
    pool_.ptr.clear();
    for (int s = 0; s < slots_; ++s) pool_.ptr.push_back(bf(expert_slot_bytes_ / 2));
    pool_.release.assign(slots_, nullptr);
    pool_.has_release.assign(slots_, 0);
    pool_.free_fifo.clear();
    for (int s = 0; s < slots_; ++s) pool_.free_fifo.push_back(s);

    norm_attn_.resize(D_.L);
    norm_ffn_.resize(D_.L);
    for (int l = 0; l < D_.L; ++l) {
        norm_attn_[l] = bf(D_.d);
        norm_ffn_[l] = bf(D_.d);
    }
    final_norm_ = bf(D_.d);
    embed_ = bf(static_cast<int64_t>(D_.V) * D_.d);
    head_ = bf(static_cast<int64_t>(D_.V) * D_.d);
    h_ = bf(t_max_ * D_.d);
    rope_tab_ = static_cast<float*>(take(tb_max_ * D_.hd * 4));  // [tb_max][hd/2] (cos, sin)
    defer_ok_ = std::getenv("KL_NO_DEFER") == nullptr;
    if (defer_possible()) {
        ypart_rows_ = static_cast<int64_t>(plan_.n_batches) * cfg_.workload.batch_size * D_.k;  // a decode step's rows
        ypart_ = static_cast<float*>(take(4 * ypart_rows_ * D_.d * 4));
    }
    if (defer_attn_possible()) {
        qkvpart_ = static_cast<float*>(take(4LL * cfg_.workload.batch_size * D_.qkv_width() * 4));
        opart_ = static_cast<float*>(take(4LL * plan_.n_batches * cfg_.workload.batch_size * D_.d * 4));
        o_deferred_.assign(static_cast<size_t>(plan_.n_batches), 0);
    }
    // Opt-in (KL_QKV_ROPE=1): bit-identical to the separate calls but no
    // faster (attention op 56.6 vs 57.1 us as a graph: the owners' epilogue
    // tail grows by what the RoPE launch cost).
    rope_fused_ok_ = std::getenv("KL_QKV_ROPE") != nullptr;
    stamp_cap_ = ops_per_step_bound(D_.L, plan_.n_batches, El_);
    stamps_dev_ = static_cast<unsigned long long*>(take((2 * stamp_cap_ + 8) * 8));
    x2_ = bf(t_max_ * D_.d);
    xa_ = bf(tb_max_ * D_.d);
    qkv_ = bf(tb_max_ * D_.qkv_width());
    ao_ = bf(tb_max_ * D_.Hq * D_.hd);
    idx_[0] = i32(R);
    idx_[1] = i32(R);
    forced_ = i32(R);
    pos_ = i32(R);
    row_token_ = i32(R);
    weight_ = static_cast<float*>(take(R * 4));
    router_logits_ = static_cast<float*>(take(t_max_ * D_.E * 4));
    const int64_t Rx = std::max<int64_t>(R, r_recv_max_);
    xp_ = bf(Rx * D_.d);
    y_ = bf(Rx * D_.d);
    hs_ = bf(std::min<int64_t>(cfg_.ffn_chunk_rows, std::max<int64_t>(Rx, 1)) * D_.f);
    if (D_.fs() > 0) hshared_ = bf(std::min<int64_t>(cfg_.ffn_chunk_rows, std::max<int64_t>(R, 1)) * D_.fs());
    perm_ws_ = take(kl_permute_workspace_bytes(Rx, D_.E));
    gemm_ws_ = gemm_ws_bytes_ > 0 ? take(gemm_ws_bytes_) : nullptr;
    tok_pos_ = i32(t_max_);
    tok_seq_ = i32(t_max_);
    tok_seq_local_ = i32(t_max_);
    ids_ = i32(t_max_);
    next_ids_ = i32(t_max_);
    last_rows_ = i32(t_max_);
    counts_ = i32(D_.E + 1);
    offsets_ = i32(D_.E + 1);
    last_h_ = bf(seqs * D_.d);
    head_logits_ = bf(seqs * D_.V);
    report_ = static_cast<int32_t*>(take(2LL * n * D_.E * 4 + 2LL * D_.E * 8 + 64));
    table_ = static_cast<int64_t*>(take((static_cast<byte_count>(std::max(D_.L - 1, 1)) * D_.E * D_.E) * 8));
    marginal_ = static_cast<int64_t*>(take(D_.E * 8));
    if (ep_) {
        label_map_ = i32(D_.E);
        lbl_ = i32(R);
        recv_ids_ = i32(r_recv_max_);
        pos2_ = i32(r_recv_max_);
        row_token2_ = i32(r_recv_max_);
        recv_counts_ = i32(D_.E);
        hist_all_ = i32(D_.E);
        counts2_ = i32(El_ + 1);
        offsets2_ = i32(El_ + 1);
        send_counts_ = i32(D_.E + 1);
        delta_ = static_cast<int64_t*>(take((static_cast<int64_t>(D_.E) * D_.E + D_.E) * 8));
        if (cfg_.ep_backend == "loopback")
            xstage_ = static_cast<int64_t*>(take(static_cast<int64_t>(G_) * (D_.E * D_.E + D_.E) * 8));
        recv_x_ = bf(r_recv_max_ * D_.d);
        y_back_ = bf(r_recv_max_ * D_.d);
        y_ret_ = bf(R * D_.d);
        std::vector<int32_t> label(D_.E);
        for (int e = 0; e < D_.E; ++e) label[e] = (e % G_) * El_ + e / G_;  // destination-major
        cuda_check(cudaMemcpy(label_map_, label.data(), D_.E * 4, cudaMemcpyHostToDevice), "label map");
    }
    const byte_count ws_real = arena_used_;

    // KV caches and resident layers (planner's decisions).
    kc_.assign(D_.L, nullptr);
    vc_.assign(D_.L, nullptr);
    if (kv_offload_) {
        // Device KV slots of one (layer, batch) each: [bs][cap][Hkv][hd] K and V.
        kv_slot_k_.clear();
        kv_slot_v_.clear();
        for (int s = 0; s < kKvSlots; ++s) {
            kv_slot_k_.push_back(static_cast<uint16_t*>(take(kv_slot_bytes_ / 2)));
            kv_slot_v_.push_back(static_cast<uint16_t*>(take(kv_slot_bytes_ / 2)));
        }
        kv_slot_release_.assign(kKvSlots, nullptr);
        kv_slot_next_ = 0;
    } else {
        for (int l = 0; l < D_.L; ++l) {
            kc_[l] = static_cast<uint16_t*>(take(kv_bytes_layer_ / 2));
            vc_[l] = static_cast<uint16_t*>(take(kv_bytes_layer_ / 2));
        }
    }
    res_expert_.assign(static_cast<size_t>(D_.L) * El_, nullptr);
    res_attn_.assign(D_.L, nullptr);
    for (int l = 0; l < D_.L; ++l) {
        if (plan_.placement.expert_tier[l] == Tier::vram)
            for (int e = 0; e < El_; ++e) res_expert_[l * El_ + e] = bf(D_.expert_elems());
        if (plan_.placement.attention_tier[l] == Tier::vram) res_attn_[l] = bf(D_.attention_elems());
    }
    if (ws_real > ws_bytes_ + 64 * 1024)
        throw AccountingError("engine: working-set estimate " + std::to_string(ws_bytes_) + " < actual " +
                              std::to_string(ws_real));
}

void Engine::allocate_host() {
    const int L = D_.L, E = El_;  // expert arrays are per local shard
    host_expert_.assign(static_cast<size_t>(L) * E, nullptr);
    host_attn_.assign(L, nullptr);
    host_gate_.assign(L, nullptr);
    // Non-resident expert layers, optionally aliased onto R distinct copies.
    // The whole-layer baseline moves every expert over the link each block
    // (its reference semantics, schedule.cpp:190-208), resident or not.
    const bool whole_layer = cfg_.variant == Variant::multibatch_full_prefetch || cfg_.variant == Variant::simple;
    std::vector<int> streamed;
    for (int l = 0; l < L; ++l)
        if ((plan_.placement.expert_tier[l] != Tier::vram || whole_layer) && plan_.placement.expert_tier[l] != Tier::disk)
            streamed.push_back(l);
    const int R = cfg_.host_distinct_layers > 0 ? std::min<int>(cfg_.host_distinct_layers, streamed.size())
                                                : static_cast<int>(streamed.size());
    std::vector<void*> blocks(R, nullptr);
    std::vector<cudaError_t> errs(R, cudaSuccess);
    const byte_count layer_bytes = expert_slot_bytes_ * E;
    {
        // Pinning is CPU-bound page work: spread it over host threads.
        std::vector<std::thread> th;
        const int workers = std::max(1, std::min<int>(8, R));
        for (int w = 0; w < workers; ++w)
            th.emplace_back([&, w] {
                for (int i = w; i < R; i += workers)
                    errs[i] = cudaHostAlloc(&blocks[i], static_cast<size_t>(layer_bytes), cudaHostAllocDefault);
            });
        for (auto& t : th) t.join();
    }
    for (int i = 0; i < R; ++i) {
        cuda_check(errs[i], "cudaHostAlloc experts");
        host_blocks_.push_back(blocks[i]);
    }
    for (size_t s = 0; s < streamed.size(); ++s) {
        char* base = static_cast<char*>(blocks[s % R]);
        for (int e = 0; e < E; ++e)
            host_expert_[streamed[s] * E + e] = reinterpret_cast<uint16_t*>(base + expert_slot_bytes_ * e);
    }
    auto pinned = [&](byte_count bytes) {
        void* p = nullptr;
        cuda_check(cudaHostAlloc(&p, static_cast<size_t>(bytes), cudaHostAllocDefault), "cudaHostAlloc");
        host_blocks_.push_back(p);
        return p;
    };
    for (int l = 0; l < L; ++l) {
        if (plan_.placement.attention_tier[l] == Tier::dram)
            host_attn_[l] = static_cast<uint16_t*>(pinned(attn_slot_bytes_));
        if (plan_.placement.gate_tier[l] != Tier::disk) host_gate_[l] = static_cast<uint16_t*>(pinned(spec_.gate_bytes));
    }
    // Disk tier: the staging window's pinned slots and the backing file.
    window_slot_of_.assign(L, -1);
    window_slot_.clear();
    window_free_.clear();
    if (plan_.placement.any_disk()) {
        const int wl = std::max(1, plan_.placement.cpu_window_L);
        for (int s = 0; s < wl; ++s) {
            window_slot_.push_back(static_cast<char*>(pinned(plan_.placement.per_layer_disk_bytes_max)));
            window_free_.push_back(s);
        }
        bounce_bytes_ = std::max({expert_slot_bytes_, attn_slot_bytes_, spec_.gate_bytes});
        for (auto& b : bounce_) b = static_cast<char*>(pinned(bounce_bytes_));
        open_disk_store();
    }
    const int n = plan_.n_batches;
    if (kv_offload_) {
        // Pinned host KV per (layer, batch): [bs][cap][Hkv][hd] K then V.
        host_kv_.assign(static_cast<size_t>(L) * n, nullptr);
        for (size_t i = 0; i < host_kv_.size(); ++i) host_kv_[i] = static_cast<uint16_t*>(pinned(kv_slot_bytes_));
    }
    stamps_host_ = static_cast<unsigned long long*>(pinned((2 * stamp_cap_ + 8) * 8));
    host_report_ = static_cast<int32_t*>(pinned(2LL * n * D_.E * 4 + 2LL * D_.E * 8 + D_.E * 4 + 128));
    if (ep_) host_recv_ids_ = static_cast<int32_t*>(pinned(std::max<int64_t>(r_recv_max_, 1) * 4));
    host_idx_ = static_cast<int32_t*>(pinned(t_max_ * D_.k * 4));
    host_forced_ = static_cast<int32_t*>(pinned(t_max_ * D_.k * 4));
    host_tokens_ = static_cast<int32_t*>(pinned(5 * t_max_ * 4));
}

void Engine::init_weights() {
    // Op end-mark counter (kl_stamp_end_next_launch): zero before first use,
    // reset by each end-marking kernel's last CTA.
    end_cnt_ = reinterpret_cast<unsigned*>(stamps_dev_ + 2 * stamp_cap_ + 4);
    cuda_check(cudaMemset(end_cnt_, 0, sizeof(unsigned)), "end counter");
    cudaStream_t st = streams_[0];
    const std::uint64_t ws = cfg_.weight_seed;
    const float sd = 0.02f;
    // Norm weights = 1.0 (bf16 0x3f80).
    std::vector<uint16_t> ones(D_.d, 0x3f80);
    for (int l = 0; l < D_.L; ++l) {
        cuda_check(cudaMemcpy(norm_attn_[l], ones.data(), D_.d * 2, cudaMemcpyHostToDevice), "norm");
        cuda_check(cudaMemcpy(norm_ffn_[l], ones.data(), D_.d * 2, cudaMemcpyHostToDevice), "norm");
    }
    cuda_check(cudaMemcpy(final_norm_, ones.data(), D_.d * 2, cudaMemcpyHostToDevice), "norm");
    kl_check(kl_fill_normal_bf16(embed_, static_cast<int64_t>(D_.V) * D_.d, tensor_seed(ws, kKindEmbed, 0, 0), 1.0f, st),
             "init embed");
    kl_check(kl_fill_normal_bf16(head_, static_cast<int64_t>(D_.V) * D_.d, tensor_seed(ws, kKindHead, 0, 0), sd, st),
             "init head");
    // Staging for host-resident tensors: a slot large enough for either kind
    // (bf16), or the bf16 scratch + a pool slot for the Q4T bytes.
    uint16_t* stage = cfg_.quant ? wscratch_
                                 : (D_.expert_elems() >= D_.attention_elems() ? pool_.ptr[0] : attn_slot_[0]);
    // The router (+ shared experts) tensor can exceed both (deepseek-v2-lite:
    // 17.4M gate elements vs 16.8M attention): it is staged in its own slot.
    uint16_t* gate_stage = gate_slot_[0];
    uint8_t* qstage = reinterpret_cast<uint8_t*>(pool_.ptr[0]);
    // bf16 experts are stored K-blocked (kl_weights_kblock: each 128-row x
    // 64-column weight tile one contiguous 16 KB run for the streaming GEMM);
    // converted from the row-major stage into a second pool slot.
    const bool kb = expert_kblocked();
    uint16_t* kb_stage = pool_.ptr[slots_ > 1 ? 1 : 0];
    if (kb && kb_stage == stage) throw AccountingError("engine: no second slot to stage K-blocked experts");
    auto kblock_expert = [&](const uint16_t* src, uint16_t* dst) {
        kl_check(kl_weights_kblock(src, 2LL * D_.f, D_.d, dst, st), "kblock w13");
        kl_check(kl_weights_kblock(src + 2LL * D_.f * D_.d, D_.d, D_.f, dst + 2LL * D_.f * D_.d, st), "kblock w2");
    };
    // bf16 stage -> host copy in the streamed format.
    auto to_host = [&](void* host, bool expert) {
        if (!cfg_.quant) {
            const uint16_t* src = stage;
            if (expert && kb) {
                kblock_expert(stage, kb_stage);
                src = kb_stage;
            }
            cuda_check(cudaMemcpyAsync(host, src, expert ? spec_.expert_bytes : spec_.attention_bytes,
                                       cudaMemcpyDeviceToHost, st), "d2h");
            return;
        }
        const int64_t r0 = expert ? 2LL * D_.f : D_.qkv_width(), k0 = D_.d;
        const int64_t r1 = D_.d, k1 = expert ? D_.f : static_cast<int64_t>(D_.Hq) * D_.hd;
        kl_check(kl_quantize_q4(stage, r0, k0, qstage, st), "quantize");
        kl_check(kl_quantize_q4(stage + r0 * k0, r1, k1, qstage + kl_q4_bytes(r0, k0), st), "quantize");
        cuda_check(cudaMemcpyAsync(host, qstage, expert ? expert_slot_bytes_ : attn_slot_bytes_, cudaMemcpyDeviceToHost, st),
                   "d2h");
    };
    std::vector<char> host_done(host_blocks_.size(), 0);
    for (int l = 0; l < D_.L; ++l) {
        // Disk-tier parts of the layer are assembled in window slot 0 (no
        // stage op has run yet) and written to the layer's file region.
        const bool on_disk = disk_fd_ >= 0 && disk_bytes(l) > 0;
        auto disk_part = [&](TensorClass cls, byte_count extra) {
            return reinterpret_cast<uint16_t*>(window_slot_[0] + disk_part_offset(l, cls) + extra);
        };
        const bool exp_disk = plan_.placement.expert_tier[l] == Tier::disk;
        uint16_t* attn_dst = plan_.placement.attention_tier[l] == Tier::disk ? disk_part(TensorClass::attention, 0)
                                                                              : host_attn_[l];
        uint16_t* gate_dst = plan_.placement.gate_tier[l] == Tier::disk ? disk_part(TensorClass::gate, 0) : host_gate_[l];
        for (int e = 0; e < El_; ++e) {
            // Seeds follow the GLOBAL expert id so every EP shard holds the
            // same weights the single-GPU engine would.
            const std::uint64_t seed = tensor_seed(ws, kKindExpert, l, ep_ ? e * G_ + rank_ : e);
            if (uint16_t* r = res_expert_[l * El_ + e]) {
                if (kb) {
                    kl_check(kl_fill_normal_bf16(stage, D_.expert_elems(), seed, sd, st), "init expert");
                    kblock_expert(stage, r);
                } else {
                    kl_check(kl_fill_normal_bf16(r, D_.expert_elems(), seed, sd, st), "init expert");
                }
                if (uint16_t* h = host_expert_[l * El_ + e]) {
                    if (cfg_.quant) {
                        cuda_check(cudaMemcpyAsync(stage, r, spec_.expert_bytes, cudaMemcpyDeviceToDevice, st), "d2d");
                        to_host(h, true);
                    } else {
                        cuda_check(cudaMemcpyAsync(h, r, spec_.expert_bytes, cudaMemcpyDeviceToHost, st), "d2h");
                    }
                }
            } else if (exp_disk) {
                kl_check(kl_fill_normal_bf16(stage, D_.expert_elems(), seed, sd, st), "init expert");
                to_host(disk_part(TensorClass::expert, expert_slot_bytes_ * e), true);
            } else if (uint16_t* h = host_expert_[l * El_ + e]) {
                // Aliased host layers are filled once, by their first user.
                bool first = true;
                for (int l2 = 0; l2 < l && first; ++l2)
                    if (host_expert_[l2 * El_ + e] == h) first = false;
                if (!first) continue;
                kl_check(kl_fill_normal_bf16(stage, D_.expert_elems(), seed, sd, st), "init expert");
                to_host(h, true);
            }
        }
        const std::uint64_t aseed = tensor_seed(ws, kKindAttn, l, 0);
        if (res_attn_[l]) {
            kl_check(kl_fill_normal_bf16(res_attn_[l], D_.attention_elems(), aseed, sd, st), "init attn");
        } else {
            kl_check(kl_fill_normal_bf16(stage, D_.attention_elems(), aseed, sd, st), "init attn");
            to_host(attn_dst, false);
        }
        kl_check(kl_fill_normal_bf16(gate_stage, D_.gate_elems(), tensor_seed(ws, kKindGate, l, 0), sd, st), "init gate");
        cuda_check(cudaMemcpyAsync(gate_dst, gate_stage, spec_.gate_bytes, cudaMemcpyDeviceToHost, st), "d2h");
        if (on_disk) {
            cuda_check(cudaStreamSynchronize(st), "init sync");
            const char* src = window_slot_[0];
            int64_t left = disk_bytes(l), off = disk_off_[l];
            while (left > 0) {
                const ssize_t w = ::pwrite(disk_fd_, src, static_cast<size_t>(left), off);
                if (w <= 0) throw moesim::DeviceError(std::string("engine: disk store write: ") + std::strerror(errno));
                src += w;
                off += w;
                left -= w;
            }
        }
    }
    // Correlation table (warm-up) and marginal to HBM.
    if (D_.L > 1)
        cuda_check(cudaMemcpyAsync(table_, table0_.counts.data(), table0_.counts.size() * 8, cudaMemcpyHostToDevice, st),
                   "table");
    cuda_check(cudaMemcpyAsync(marginal_, table0_.marginal.data(), D_.E * 8, cudaMemcpyHostToDevice, st), "marginal");
    cuda_check(cudaMemsetAsync(h_, 0, t_max_ * D_.d * 2, st), "h");
    // A decode step fed from the device reads the previous step's greedy ids;
    // before any step has produced them they are token 0, never garbage.
    cuda_check(cudaMemsetAsync(next_ids_, 0, t_max_ * 4, st), "next ids");
    cuda_check(cudaStreamSynchronize(st), "init sync");
    (void)host_done;
}

void Engine::fill_kv_synthetic(int positions, std::uint64_t seed) {
    if (cfg_.plan_only) throw ConfigError("engine: created with plan_only (no KV cache)");
    // KV content of a synthetic prefill: values for the retained slots of
    // positions [0, positions) of every sequence (post-rope keys are just
    // random vectors here; the decode kernels read them like real ones).
    cudaStream_t st = streams_[0];
    const int64_t per_seq = static_cast<int64_t>(kv_cap_) * D_.Hkv * D_.hd;
    const int64_t seqs = static_cast<int64_t>(cfg_.workload.batch_size) * plan_.n_batches;
    const int filled = std::min(positions, kv_cap_);
    if (kv_offload_) {
        for (int l = 0; l < D_.L; ++l)
            for (int b = 0; b < plan_.n_batches; ++b) {
                const int64_t half = kv_slot_bytes_ / 2 / 2;  // elements of K (or V)
                kl_check(kl_fill_normal_bf16(kv_slot_k_[0], half, mix64(seed, 2 * (l * plan_.n_batches + b)), 1.0f, st),
                         "kv fill");
                kl_check(kl_fill_normal_bf16(kv_slot_v_[0], half, mix64(seed, 2 * (l * plan_.n_batches + b) + 1), 1.0f,
                                             st), "kv fill");
                uint16_t* h = host_kv_[static_cast<size_t>(l) * plan_.n_batches + b];
                cuda_check(cudaMemcpyAsync(h, kv_slot_k_[0], kv_slot_bytes_ / 2, cudaMemcpyDeviceToHost, st), "kv d2h");
                cuda_check(cudaMemcpyAsync(h + half, kv_slot_v_[0], kv_slot_bytes_ / 2, cudaMemcpyDeviceToHost, st), "kv d2h");
            }
        cuda_check(cudaStreamSynchronize(st), "kv fill sync");
        kv_filled_positions_ = filled;
        return;
    }
    for (int l = 0; l < D_.L; ++l) {
        // Whole-cache fill (unused slots are never read: attention reads
        // min(pos+1, cap) slots).
        kl_check(kl_fill_normal_bf16(kc_[l], per_seq * seqs, mix64(seed, 2 * l), 1.0f, st), "kv fill");
        kl_check(kl_fill_normal_bf16(vc_[l], per_seq * seqs, mix64(seed, 2 * l + 1), 1.0f, st), "kv fill");
    }
    (void)filled;
    cuda_check(cudaStreamSynchronize(st), "kv fill sync");
}

std::string Engine::describe() const {
    json j;
    j["plan_text"] = plan_.to_text();
    j["n_batches"] = plan_.n_batches;
    j["solved_n_uncapped"] = plan_.solved_n_uncapped;
    j["planner_solved_n"] = planner_solved_n_;       // reference working-set model, before the KV cap
    j["planner_n"] = planner_n_;                     // ... after its KV cap
    j["memory_capped_n"] = memory_capped_n_;         // 0 = the engine's working set did not cap n
    j["kv_capped"] = plan_.kv_capped;
    j["batch_size"] = cfg_.workload.batch_size;
    j["prompt_len"] = cfg_.workload.prompt_len;
    j["gen_len"] = cfg_.workload.gen_len;
    j["expert_slots"] = slots_;
    j["arena_used_bytes"] = arena_used_;
    j["hbm_cap_bytes"] = cfg_.hbm_cap;
    j["working_set_bytes"] = ws_bytes_;
    j["kv_cap_tokens"] = kv_cap_;
    j["kv_sink"] = kv_sink_;
    j["kv_bytes_per_layer"] = kv_bytes_layer_;
    j["kv_offload"] = kv_offload_;
    j["kv_slot_bytes"] = kv_slot_bytes_;
    int resident = 0, attn_res = 0;
    for (int l = 0; l < D_.L; ++l) {
        resident += plan_.placement.expert_tier[l] == Tier::vram;
        attn_res += plan_.placement.attention_tier[l] == Tier::vram;
    }
    j["resident_expert_layers"] = resident;
    {
        std::vector<int> et, at;
        for (int l = 0; l < D_.L; ++l) {
            et.push_back(plan_.placement.expert_tier[l] == Tier::vram ? 1 : 0);
            at.push_back(plan_.placement.attention_tier[l] == Tier::vram ? 1 : 0);
        }
        j["expert_resident"] = et;
        j["attention_resident"] = at;
    }
    j["resident_attention_layers"] = attn_res;
    j["expert_bytes"] = spec_.expert_bytes;
    j["attention_bytes"] = spec_.attention_bytes;
    j["expert_stream_bytes"] = expert_slot_bytes_;
    j["attention_stream_bytes"] = attn_slot_bytes_;
    j["quant_bits"] = cfg_.quant ? cfg_.quant->bits : 16;
    j["expert_layout"] = expert_kblocked() ? "kblocked" : (cfg_.quant ? "q4t" : "row");
    j["gate_bytes"] = spec_.gate_bytes;
    j["shared_experts"] = {{"n", D_.n_shared}, {"f", D_.f_shared}};
    j["host_pinned_blocks"] = host_blocks_.size();
    {
        std::vector<int> dl;
        for (int l = 0; l < D_.L; ++l) dl.push_back(plan_.placement.disk_bytes_of_layer(l, spec_, cfg_.quant) > 0 ? 1 : 0);
        j["disk_layers"] = dl;
        j["cpu_window_L"] = plan_.placement.cpu_window_L;
        j["disk_store_bytes"] = disk_bytes_total_;
        j["window_slot_bytes"] = plan_.placement.per_layer_disk_bytes_max;
    }
    // Everything needed to rebuild the same plan/schedule with the reference.
    j["spec"] = {{"n_layers", spec_.n_layers}, {"n_experts", spec_.n_experts_per_layer}, {"top_k", spec_.top_k},
                 {"expert_bytes", spec_.expert_bytes}, {"attention_bytes", spec_.attention_bytes},
                 {"gate_bytes", spec_.gate_bytes}, {"kv_bytes_per_token", spec_.kv_bytes_per_token}};
    j["profile"] = {{"vram_capacity", profile_.vram_capacity}, {"dram_capacity", profile_.dram_capacity},
                    {"disk_capacity", profile_.disk_capacity}, {"pcie_bandwidth", profile_.pcie_bandwidth},
                    {"disk_bandwidth", profile_.disk_bandwidth}, {"transfer_fixed_latency_ps", 0},
                    {"attn_ps", profile_.attn_compute_per_token}, {"gate_ps", profile_.gate_compute_per_token},
                    {"expert_ps", profile_.expert_compute_per_token}};
    if (measured_) j["measured_profile"] = json::parse(measured_->to_json());
    j["streaming_kv"] = cfg_.retention.mode == KvRetentionPolicy::Mode::streaming;
    j["sink_tokens"] = cfg_.retention.sink_tokens;
    j["window_tokens"] = cfg_.retention.window_tokens;
    j["dims"] = {{"L", D_.L}, {"d", D_.d}, {"f", D_.f}, {"Hq", D_.Hq}, {"Hkv", D_.Hkv}, {"hd", D_.hd},
                 {"E", D_.E}, {"k", D_.k}, {"V", D_.V}, {"theta", D_.theta}, {"eps", D_.eps},
                 {"score_mode", D_.score_mode}, {"n_shared", D_.n_shared}, {"f_shared", D_.f_shared}};
    return j.dump();
}

}  // namespace klotski
