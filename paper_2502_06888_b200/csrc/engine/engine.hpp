// SPDX-License-Identifier: Apache-2.0
// B200 execution engine for the Klotski pipeline (internal header).
//
// Drives the reference's Algorithm 1 online (detail::Emitter, shared with
// moesim::build_klotski_schedule) and executes each emitted StreamOp:
//   load_weights / load_expert -> cudaMemcpyAsync H2D from pinned host into
//                                 the attention / gate / expert slot pools
//   compute_attention          -> rmsnorm + tcgen05 QKV GEMM + rope/KV append
//                                 + decode|prefill attention + O GEMM(+resid)
//   compute_gate               -> fused rmsnorm/router/top-k (+ at the last
//                                 gate: permute, co-activation update,
//                                 next-layer prefetch scores, routing readback)
//   compute_expert             -> SwiGLU expert FFN on the expert's rows
//                                 (+ combine after the block's last expert)
//   offload_*                  -> slot release by event (no bytes move)
// Streams mirror moesim::StreamId; dependencies are cudaEvents; the
// timeline is measured with events and reduced with the reference metrics.
#pragma once

#include <cuda_runtime_api.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "../host/emitter.hpp"
#include "moesim/quant.hpp"
#include "moesim/experiment.hpp"
#include "moesim/simulator.hpp"

namespace klotski {


using moesim::byte_count;

struct Dims {
    int L = 4, d = 512, f = 1792, Hq = 8, Hkv = 2, hd = 64, E = 8, k = 2, V = 1024;
    float theta = 1e6f, eps = 1e-5f;
    int score_mode = 0;
    // Shared (always-active) experts, e.g. DeepSeek-V2-Lite's 2 x 1408. They
    // are one SwiGLU FFN of intermediate n_shared * f_shared on every token,
    // streamed with the router as the dense part of the MoE layer (an
    // additive extension: the reference ModelSpec has no such field, so they
    // are accounted in gate_bytes).
    int n_shared = 0, f_shared = 0;
    int fs() const { return n_shared * f_shared; }
    byte_count shared_elems() const { return 3LL * d * fs(); }
    int qkv_width() const { return (Hq + 2 * Hkv) * hd; }
    byte_count expert_elems() const { return 3LL * d * f; }
    byte_count attention_elems() const { return static_cast<byte_count>(qkv_width()) * d + static_cast<byte_count>(d) * Hq * hd; }
    byte_count gate_elems() const { return static_cast<byte_count>(E) * d + shared_elems(); }
};

struct EngineConfig {
    Dims dims;
    std::string name = "tiny";
    moesim::BatchGroupConfig workload;
    moesim::KvRetentionPolicy retention;
    byte_count hbm_cap = 24'000'000'000LL;
    byte_count host_dram = 190'000'000'000LL;
    double pcie_bandwidth = 55.0e9;
    moesim::duration_ps attn_ps = 1'000'000, gate_ps = 20'000, expert_ps = 300'000;
    std::optional<int> n_override;
    moesim::Variant variant = moesim::Variant::klotski;
    bool replay = false;
    moesim::SkewSpec skew = moesim::SkewSpec::zipf(1.5);
    std::uint64_t trace_seed = 1, warmup_seed = 0, weight_seed = 7;
    int host_distinct_layers = 0;
    int expert_slots = 0;
    int ffn_chunk_rows = 4096;
    bool kblocked_experts = true;  // bf16 experts stored K-blocked (kl_weights_kblock); Q4T keeps its own tiles
    bool record_trace = true;
    bool record_hidden = false;
    int ep_rank = 0, ep_world = 1;
    bool ep = false;                // expert-parallel engine (also for world 1)
    std::string ep_nccl_id;         // 256 hex chars of ncclUniqueId (world > 1, backend nccl)
    // Exchange backend for world > 1: "nccl" (one process per GPU) or
    // "loopback" (G engines of one process on one device, host threads,
    // device copies + events; rendezvous by ep_group name).
    std::string ep_backend = "nccl";
    std::string ep_group;
    bool prefill = true;
    bool plan_only = false;  // stop after planning (describe() only): n, placement, working set
    std::optional<moesim::QuantConfig> quant;  // 4-bit streamed experts / attention (Q4T)
    std::string disk_dir;           // disk-tier store directory (default $TMPDIR, else /tmp)
    std::string measure_phase;      // "decode" | "prefill": plan with rates measured on this GPU
};

EngineConfig parse_config(const std::string& json_text);

// Planner stage 1 (engine_profile.cpp): this engine's kernels and the pinned
// host link timed on the model's shapes -> HardwareProfile rates.
struct MeasuredProfile {
    std::string phase;
    int tokens_per_batch = 0, expert_rows = 0, kv_slots = 0;
    double attn_ms = 0, gate_ms = 0, expert_ms = 0, h2d_1_gbs = 0, h2d_2_gbs = 0;
    moesim::duration_ps attn_ps = 0, gate_ps = 0, expert_ps = 0;
    double pcie_bandwidth = 0;
    std::string to_json() const;
};
MeasuredProfile measure_profile(const EngineConfig& cfg, const std::string& phase);

struct ExpertSlotPool {
    std::vector<uint16_t*> ptr;
    std::vector<cudaEvent_t> release;     // valid when has_release
    std::vector<char> has_release;
    std::deque<int> free_fifo;            // least recently released first
    int acquire();
    void release_after(int slot, cudaEvent_t ev);
};

class Engine {
  public:
    explicit Engine(const EngineConfig& cfg);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void fill_kv_synthetic(int positions, std::uint64_t seed);
    double step(int step, const int32_t* tokens_in, int32_t* next_out);
    std::string describe() const;
    std::string report(const std::string& what);
    void reset_log();
    void read_hidden(uint16_t* host, int64_t n) const;
    struct Exchange;  // expert-parallel exchange backend (engine_ep.cpp)

  private:
    // setup
    void plan_memory();
    bool expert_kblocked() const { return cfg_.kblocked_experts && !cfg_.quant; }
    bool plan_at(int n, bool rethrow = false);
    void finish_plan();
    moesim::TraceStats stats_;
    int planner_solved_n_ = 0, planner_n_ = 0, memory_capped_n_ = 0;
    void allocate_device();
    void allocate_host();
    void init_weights();
    void* take(byte_count bytes);

    // execution
    void issue_pending();
    void exec(std::int32_t id);
    void exec_attention(const moesim::StreamOp& op);
    void exec_gate(const moesim::StreamOp& op);
    void exec_expert(const moesim::StreamOp& op);
    void combine_block(int step);
    int combine_step_ = -1;
    void after_layer_gates(int step, int layer);
    moesim::detail::BlockRouting read_routing(int step, int layer);
    moesim::PrefetchDecision decide(int step, int layer) const;
    cudaStream_t stream_of(moesim::StreamId s) const { return streams_[static_cast<int>(s)]; }
    cudaEvent_t event();
    void collect_step_times();
    int tokens_per_batch(int step) const { return cfg_.workload.batch_size * (step == 0 ? cfg_.workload.prompt_len : 1); }
    int n_batches() const { return plan_.n_batches; }
    const uint16_t* expert_weights(int layer, int e) const;

    EngineConfig cfg_;
    Dims D_;
    moesim::ModelSpec spec_;
    moesim::HardwareProfile profile_;
    std::optional<MeasuredProfile> measured_;
    moesim::PipelinePlan plan_;
    moesim::CorrelationTable table0_;
    moesim::ActivationTrace replay_trace_;
    moesim::ActivationTrace recorded_;
    std::unique_ptr<moesim::detail::Emitter> em_;
    std::int32_t next_exec_ = 0;

    // memory plan
    byte_count ws_bytes_ = 0, kv_bytes_layer_ = 0;
    int kv_cap_ = 0, kv_sink_ = 0;
    int64_t t_max_ = 0, tb_max_ = 0;
    int slots_ = 0;
    char* arena_ = nullptr;
    byte_count arena_used_ = 0;

    // device buffers
    std::vector<uint16_t*> res_expert_;  // [L*E] resident expert weights (or null)
    std::vector<uint16_t*> res_attn_;    // [L]
    std::vector<uint16_t*> norm_attn_, norm_ffn_;
    uint16_t* final_norm_ = nullptr;
    uint16_t *embed_ = nullptr, *head_ = nullptr;
    std::vector<uint16_t*> kc_, vc_;     // [L]
    uint16_t *h_ = nullptr, *x2_ = nullptr, *xa_ = nullptr, *qkv_ = nullptr, *ao_ = nullptr;
    uint16_t *xp_ = nullptr, *y_ = nullptr, *hs_ = nullptr, *last_h_ = nullptr, *head_logits_ = nullptr;
    uint16_t* hshared_ = nullptr;  // shared-expert SwiGLU output, [chunk rows][fs]
    void shared_experts(int layer, int64_t T, int64_t row0);
    void after_batch_gate(int step, int layer, int b);
    moesim::detail::BlockRouting read_routing_row(int step, int layer, int b);
    int combine_batch_ = -1;
    int32_t *idx_[2] = {nullptr, nullptr}, *forced_ = nullptr, *pos_ = nullptr, *row_token_ = nullptr;
    int32_t *counts_ = nullptr, *offsets_ = nullptr, *tok_pos_ = nullptr, *tok_seq_ = nullptr;
    int32_t *ids_ = nullptr, *next_ids_ = nullptr, *last_rows_ = nullptr;
    float *weight_ = nullptr, *router_logits_ = nullptr;
    void* perm_ws_ = nullptr;
    void* gemm_ws_ = nullptr;            // split-K fp32 partials (decode GEMMs)
    int64_t gemm_ws_bytes_ = 0;
    int32_t* report_ = nullptr;          // [n*E hist | n*E first] + int64 [E scores | E marginal]
    int64_t *table_ = nullptr, *marginal_ = nullptr;
    std::vector<uint16_t*> attn_slot_, gate_slot_;
    ExpertSlotPool pool_;

    // host (pinned) store
    std::vector<void*> host_blocks_;
    std::vector<uint16_t*> host_expert_;  // [L*E] (null when resident); Q4T bytes when quantised
    byte_count expert_slot_bytes_ = 0;    // bytes of a streamed expert (bf16, or Q4T = plan.cost.expert_transfer_bytes)
    byte_count attn_slot_bytes_ = 0;      // bytes of streamed attention weights (bf16 or Q4T)
    uint16_t* wscratch_ = nullptr;        // Q4: bf16 staging / dequantised weights for M > 256
    std::vector<uint16_t*> host_attn_;    // [L]
    std::vector<uint16_t*> host_gate_;    // [L]

    // Disk tier + DRAM staging window (placement.cpp window_advance,
    // schedule.cpp advance_window / stage_prologue): disk-resident tensors of
    // a layer live in one unlinked file region [experts | gate | attention]
    // (only the disk-tier parts, in streamed format); window_stage ops read a
    // layer's region into one of cpu_window_L pinned window slots with pread
    // from a host function on the cpu_stage stream, and that layer's H2D
    // loads take their source from the slot.
    struct StageJob {
        Engine* eng;
        char* dst;
        int64_t off, bytes;
    };
    int disk_fd_ = -1;
    std::vector<int64_t> disk_off_;       // [L] file offset of the layer's region
    std::vector<char*> window_slot_;      // [cpu_window_L] pinned, per_layer_disk_bytes_max each
    std::vector<int> window_slot_of_;     // [L] slot holding the layer (emission order), -1 none
    std::deque<int> window_free_;
    std::array<char*, 2> bounce_{};       // per load stream: direct reads of unstaged disk tensors
    byte_count bounce_bytes_ = 0;
    std::deque<StageJob> stage_jobs_;     // stable addresses for in-flight host functions
    std::atomic<int> stage_errno_{0};
    std::atomic<int64_t> disk_bytes_read_{0};
    int64_t disk_bytes_total_ = 0, direct_reads_ = 0, direct_bytes_ = 0;
    byte_count disk_bytes(int layer) const;
    byte_count disk_part_offset(int layer, moesim::TensorClass cls) const;
    // Host source of a streamed tensor for an H2D load enqueued on `st`.
    const void* load_src(moesim::TensorClass cls, int layer, int e, cudaStream_t st);
    void enqueue_disk_read(char* dst, int64_t off, int64_t bytes, cudaStream_t st);
    void open_disk_store();
    void stage_read(const StageJob& job);
    static void CUDART_CB stage_host_fn(void* job);
    int32_t* host_report_ = nullptr;
    int32_t* host_idx_ = nullptr;
    int32_t* host_tokens_ = nullptr;
    int32_t* host_forced_ = nullptr;

    // streams / events
    std::array<cudaStream_t, moesim::kNumStreams> streams_{};
    // Dependency / release events (cudaEventDisableTiming: recording one is
    // free even while a copy engine streams, unlike a timed event). Two pools
    // alternate by step so a step never reuses an event the previous one
    // may still reference.
    std::array<std::vector<cudaEvent_t>, 2> event_pool_;
    int event_par_ = 0;
    std::size_t event_next_ = 0;
    cudaEvent_t step_begin_ = nullptr, step_end_ = nullptr;  // timed: one pair per step
    // Op timing: device timestamps (kl_stamp, GPU global timer in ns) at each
    // op's start and end, indexed by op id - timed_from_; read back once the
    // step has synchronized. [0, 2*cap): the window's stamps; [2*cap]: t0.
    unsigned long long* stamps_dev_ = nullptr;
    unsigned long long* stamps_host_ = nullptr;
    std::int64_t stamp_cap_ = 0;  // ops per step window
    bool t0_recorded_ = false;
    unsigned long long t0_ns_ = 0;
    void stamp(std::int32_t id, int side, cudaStream_t st);
    void stamp_next_launch(std::int32_t id);  // the op's first GEMM writes its start mark
    std::vector<cudaEvent_t> op_end_;                 // by op id (current step window)
    float* rope_tab_ = nullptr;   // decode RoPE (cos, sin) table of one batch [tb_max][hd/2][2]
    // Deferred down-projection reduction (decode, bf16 K-blocked experts):
    // the split partials of every expert of a block [4][ypart_rows_][d] fp32,
    // summed by kl_combine_deferred. block_defer_ = their split count for the
    // block being executed (0 = plain kl_expert_ffn_kb + kl_combine).
    float* qkvpart_ = nullptr;    // deferred QKV split partials of one decode batch [4][bs][qkv_width]
    float* opart_ = nullptr;      // deferred o-proj split partials per batch [n][4][bs][d], summed by the gate
    int o_defer_ = -1;            // split count of the decode o-proj (-1: not yet queried, 0: off)
    std::vector<int> o_deferred_; // per batch: its o-proj partials await the gate (split count, 0 = none)
    int qkv_defer_ = -1;          // split count of the decode QKV GEMM (-1: not yet queried, 0: off)
    float* ypart_ = nullptr;
    int64_t ypart_rows_ = 0;
    bool defer_ok_ = false;
    int block_defer_ = 0;
    bool defer_possible() const;       // FFN down projection -> combine
    bool defer_attn_possible() const;  // QKV -> RoPE kernel, o-projection -> router kernel
    int block_defer_splits(std::int32_t first_op) const;
    bool rope_fused_ok_ = true;   // QKV GEMM with the fused RoPE / KV-append epilogue
    std::vector<moesim::SimEvent> timeline_;          // measured, by op id
    std::int32_t timed_from_ = 0;
    std::int32_t log_from_ = 0;
    size_t records_from_ = 0;

    // per-block execution state
    int cur_step_ = -1;
    // KV offload (KV tier = DRAM, reference load_cache / store_cache ops).
    bool kv_offload_ = false;
    byte_count kv_slot_bytes_ = 0;                 // one (layer, batch): K + V
    std::vector<uint16_t*> host_kv_;               // [L * n] pinned, K then V
    std::vector<uint16_t*> kv_slot_k_, kv_slot_v_; // device slots
    std::vector<cudaEvent_t> kv_slot_release_;     // after the slot's store
    int kv_slot_next_ = 0;
    std::map<std::pair<int, int>, int> kv_slot_of_;  // (layer, batch) -> slot
    int32_t* tok_seq_local_ = nullptr;             // row -> sequence within its batch
    int kv_filled_positions_ = 0;
    int acquire_kv_slot(cudaStream_t st);
    std::set<int> executed_steps_;
    int idx_cur_ = 0;
    std::map<std::pair<int, int>, int> expert_slot_of_;   // (layer, e) -> pool slot
    std::map<int, int> attn_slot_of_;                      // layer -> attention slot
    std::map<int, int> gate_slot_of_;                      // layer -> gate slot
    std::map<int, std::vector<int>> moe_slots_of_;         // layer -> pool slots (baselines)
    std::vector<int> attn_slot_busy_, gate_slot_busy_;
    std::vector<cudaEvent_t> attn_slot_release_, gate_slot_release_;
    std::vector<int64_t> row_offset_;                      // expert segment starts (block)
    std::vector<std::vector<int64_t>> batch_prefix_;       // [b][e] rows before batch b in e's segment
    int64_t block_rows_ = 0;
    int block_layer_ = -1;
    int exec_expert_left_ = 0;
    std::vector<int64_t> host_scores_, host_marginal_;
    // Routing readback in two parts (non-EP blocks): the per-batch histogram /
    // first demand (and recorded ids) right after the last gate, so the host
    // emits the expert half while the GPU permutes; the prefetcher's next-layer
    // scores with the rest of the op, read before the next block's decision.
    // Both parts are copied on their own stream (rb_stream_), behind events
    // recorded on the compute stream, so the compute stream never waits for
    // a PCIe round trip; the next block's first histogram reset waits for
    // readback_done_ before it rewrites the device report.
    cudaStream_t rb_stream_ = nullptr;
    cudaEvent_t routing_ready_ = nullptr, gates_done_ = nullptr, scores_done_ = nullptr, scores_ready_ = nullptr;
    std::int32_t start_mark_ = -1;  // op whose start the next kernel writes (take_start_mark before it)
    // Op end written by the op's last kernel (end_mark_next right before it);
    // exec() falls back to a stamp kernel when no launch took the mark.
    std::int32_t cur_op_ = -1;
    bool end_set_ = false;
    unsigned* end_cnt_ = nullptr;
    void end_mark_next();
    void take_start_mark();
    bool scores_pending_ = false;   // a scores readback is in flight (take_scores syncs scores_ready_)
    bool readback_pending_ = false;  // scores_ready_ recorded and not yet waited for by the compute stream
    void take_scores();
    bool scores_valid_ = false;
    int64_t tokens_generated_ = 0;
    int64_t launches_ = 0;  // sm_100a kernel launches since the last reset

    // ---- expert parallelism (engine_ep.cpp) ----
    // Global expert e lives on rank e % G as local expert e / G. Each rank
    // runs attention + router for its own batch group, streams only its
    // expert shard, and exchanges routed rows with NCCL all-to-all.
    void ep_init();
    void ep_after_gates(int step, int layer);
    moesim::detail::BlockRouting ep_read_routing(int step, int layer);
    void ep_dispatch();
    void ep_return(int64_t T);
    void exchange_rows(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& scnt, char* recv,
                       const std::vector<int64_t>& roff, const std::vector<int64_t>& rcnt, int64_t row_bytes,
                       cudaStream_t st);
    moesim::ModelSpec spec_g_;            // global model (E experts) for traces/tables
    bool ep_ = false;
    int G_ = 1, rank_ = 0, El_ = 0;
    Exchange* xch_ = nullptr;
    int64_t* xstage_ = nullptr;           // loopback all-reduce staging, [G][E*E + E] int64
    void ep_shutdown();
    int32_t *label_map_ = nullptr, *lbl_ = nullptr, *recv_ids_ = nullptr, *pos2_ = nullptr, *row_token2_ = nullptr;
    int32_t *recv_counts_ = nullptr, *hist_all_ = nullptr, *counts2_ = nullptr, *offsets2_ = nullptr;
    int32_t *send_counts_ = nullptr;
    int64_t* delta_ = nullptr;
    uint16_t *recv_x_ = nullptr, *y_back_ = nullptr, *y_ret_ = nullptr;
    int64_t r_recv_max_ = 0, r_recv_ = 0, r_send_ = 0;
    int64_t ep_max_local_rows_ = 0;       // most rows one local expert received (since reset)
    std::vector<int64_t> send_cnt_, send_off_, recv_cnt_, recv_off_;
    int32_t* host_recv_ids_ = nullptr;
    bool dispatched_ = false;
    std::vector<std::vector<uint16_t>> hidden_dumps_;
    std::vector<double> step_ms_;
};

}  // namespace klotski
