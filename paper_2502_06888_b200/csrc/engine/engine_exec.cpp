// SPDX-License-Identifier: Apache-2.0
// B200 execution engine: per-step / per-block driver and per-op execution.
//
// For each (step, layer) block the host
//   1. derives the prefetch decision from the device-side co-activation
//      table (make_table_prefetcher semantics, schedule.cpp:60-91),
//   2. emits Algorithm-1's first half (Emitter::open_block) and enqueues it:
//      gate + hot expert H2D on the weight_load stream overlapping this
//      block's n attentions (Eq. 2), n gate kernels,
//   3. waits for the routing readback of the last gate (tiny D2H),
//   4. emits the second half (cold loads in first-demand order on the
//      expert_load stream, expert computes hot-first, immediate offloads)
//      and enqueues it.
// Every op records start/end cudaEvents; cross-stream deps are
// cudaStreamWaitEvent; expert slots are reused only after the release event
// of their previous occupant (bounded pool with backpressure).
#include <limits>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <stdexcept>

#include <nlohmann/json.hpp>
#include <nvtx3/nvToolsExt.h>

#include "engine.hpp"
#include "klotski/kernels.h"
#include "metrics.hpp"

namespace klotski {

using json = nlohmann::json;
using namespace moesim;

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw moesim::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
void kl_check_impl(int rc, const char* what) {
    if (rc != 0) throw moesim::DeviceError(std::string(what) + ": " + kl_error_string(rc));
}
// Every kernel entry point goes through here (inside Engine members), which
// also counts launches for the bench's gpu_launches claim.
#define kl_check(rc, what) (++launches_, kl_check_impl((rc), (what)))

// NVTX3 range over a host-side scope: one per step and one per
// executed op, named by the op kind, so an nsys / ncu --nvtx capture shows the
// engine's enqueue structure over the kernels. A no-op without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int32_t kNoPos = 0x7f7f7f7f;  // memset(0x7f) sentinel for first_pos

// The reference's RunMetrics / bubble_stats (simulator.cpp:256-331) over one
// window of a timeline (measured or simulated), makespan counted from the
// window's first op.
json reference_metrics(const Schedule& s, size_t records_from, const std::vector<SimEvent>& tl, byte_count peak_vram,
                       int64_t tokens) {
    json j;
    Schedule view;
    view.batch_size = s.batch_size;
    view.n_batches = s.n_batches;
    view.n_steps = s.n_steps;
    view.ops = s.ops;
    view.prefetch_records.assign(s.prefetch_records.begin() + records_from, s.prefetch_records.end());
    RunMetrics m;
    detail::finalize_metrics(view, tl, peak_vram, m);
    duration_ps t_begin = tl.empty() ? 0 : tl.front().start;
    for (const SimEvent& e : tl) t_begin = std::min(t_begin, e.start);
    m.makespan -= t_begin;  // measured from the first op of the window
    m.bubble_time = m.makespan - m.compute_busy;
    m.tokens_generated = tokens;
    m.throughput_tps = m.makespan > 0 ? static_cast<double>(tokens) / sec_from_ps(m.makespan) : 0.0;
    j["makespan_ps"] = m.makespan;
    j["compute_busy_ps"] = m.compute_busy;
    j["bubble_ps"] = m.bubble_time;
    j["bubble_fraction"] = m.makespan > 0 ? static_cast<double>(m.bubble_time) / m.makespan : 0.0;
    j["expert_layer_bubble_ps"] = m.expert_layer_bubble_time;
    j["throughput_tps"] = m.throughput_tps;
    j["tokens_generated"] = m.tokens_generated;
    j["peak_vram_bytes"] = m.peak_vram;
    j["prefetch_participation"] = m.prefetch_participation;
    j["hot_accuracy"] = m.hot_accuracy;
    const BubbleBreakdown& b = m.bubbles;
    j["bubbles_ps"] = {{"startup", b.startup - t_begin},    {"intra_attention", b.intra_attention},
                       {"attn_to_moe", b.attn_to_moe},      {"intra_gate", b.intra_gate},
                       {"gate_to_expert", b.gate_to_expert}, {"intra_expert", b.intra_expert},
                       {"moe_to_attn", b.moe_to_attn},      {"drain", b.drain}};
    return j;
}

// Bytes moved by load ops and the time the host link had at least one load
// in flight (union of the load intervals).
std::pair<int64_t, duration_ps> link_usage(const Schedule& s, const std::vector<SimEvent>& tl) {
    std::vector<std::pair<duration_ps, duration_ps>> iv;
    int64_t h2d = 0;
    for (const SimEvent& e : tl) {
        const StreamOp& op = s.ops[e.op_id];
        if (op.kind == OpKind::load_weights || op.kind == OpKind::load_expert) {
            h2d += op.payload_bytes;
            iv.emplace_back(e.start, e.end);
        }
    }
    std::sort(iv.begin(), iv.end());
    duration_ps busy = 0, cur_s = -1, cur_e = -1;
    for (const auto& [a, bnd] : iv) {
        if (a > cur_e) {
            if (cur_e > cur_s) busy += cur_e - cur_s;
            cur_s = a;
            cur_e = bnd;
        } else {
            cur_e = std::max(cur_e, bnd);
        }
    }
    if (cur_e > cur_s) busy += cur_e - cur_s;
    return {h2d, busy};
}

}  // namespace


cudaEvent_t Engine::event() {
    auto& pool = event_pool_[event_par_];
    if (event_next_ == pool.size()) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        pool.push_back(e);
    }
    return pool[event_next_++];
}

// Op boundary timestamp on the op's own stream (kl_stamp).
void Engine::stamp(std::int32_t id, int side, cudaStream_t st) {
    const std::int64_t slot = static_cast<std::int64_t>(id) - timed_from_;
    if (slot < 0 || slot >= stamp_cap_)
        throw AccountingError("engine: op " + std::to_string(id) + " outside the step's timestamp window (" +
                              std::to_string(stamp_cap_) + " ops)");
    static const bool off = std::getenv("KL_PROBE_NO_STAMPS") != nullptr;  // overhead probe only: no timeline
    if (off) return;
    kl_check(kl_stamp(stamps_dev_ + 2 * slot + side, st), "op stamp");
}

// The op whose start mark the next kernel launch writes (set by exec()).
void Engine::take_start_mark() {
    if (start_mark_ < 0) return;
    stamp_next_launch(start_mark_);
    start_mark_ = -1;
}

void Engine::end_mark_next() {
    const std::int64_t slot = static_cast<std::int64_t>(cur_op_) - timed_from_;
    if (slot < 0 || slot >= stamp_cap_) return;  // exec() then stamps (and reports the window error)
    kl_check(kl_stamp_end_next_launch(stamps_dev_ + 2 * slot + 1, end_cnt_), "end mark");
    end_set_ = true;
}

void Engine::stamp_next_launch(std::int32_t id) {
    const std::int64_t slot = static_cast<std::int64_t>(id) - timed_from_;
    if (slot < 0 || slot >= stamp_cap_)
        throw AccountingError("engine: op " + std::to_string(id) + " outside the step's timestamp window");
    kl_stamp_next_launch(stamps_dev_ + 2 * slot);
}

const uint16_t* Engine::expert_weights(int layer, int e) const {
    if (const uint16_t* r = res_expert_[static_cast<size_t>(layer) * El_ + e]) return r;
    const auto it = expert_slot_of_.find({layer, e});
    if (it == expert_slot_of_.end())
        throw AccountingError("engine: expert (" + std::to_string(layer) + "," + std::to_string(e) +
                              ") computed without a loaded slot");
    return pool_.ptr[it->second];
}

int Engine::acquire_kv_slot(cudaStream_t st) {
    const int s = kv_slot_next_;
    kv_slot_next_ = (kv_slot_next_ + 1) % static_cast<int>(kv_slot_k_.size());
    for (const auto& [key, slot] : kv_slot_of_)
        if (slot == s) throw AccountingError("engine: KV slot reused before its store (raise kKvSlots)");
    if (kv_slot_release_[s] != nullptr) cuda_check(cudaStreamWaitEvent(st, kv_slot_release_[s], 0), "kv slot wait");
    return s;
}

PrefetchDecision Engine::decide(int /*step*/, int layer) const {
    PrefetchDecision d;
    d.layer = layer;
    std::vector<int64_t> score;
    if (layer == 0) {
        score = host_marginal_;
        d.used_fallback = true;
    } else {
        score = host_scores_;
        if (std::all_of(score.begin(), score.end(), [](int64_t v) { return v == 0; })) {
            score = host_marginal_;
            d.used_fallback = true;
        }
    }
    // Candidates are this rank's experts (all of them without EP): local id
    // j is global expert j*G + rank; ties keep the lower id (correlation.cpp:75-84).
    std::vector<int> ids(El_);
    std::iota(ids.begin(), ids.end(), 0);
    auto sc = [&](int j) { return score[static_cast<size_t>(j) * G_ + rank_]; };
    std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return sc(a) != sc(b) ? sc(a) > sc(b) : a < b; });
    ids.resize(std::min(spec_.top_k, El_));
    d.expert_ids = ids;
    for (int id : ids) d.scores.push_back(sc(id));
    return d;
}

double Engine::step(int step, const int32_t* tokens_in, int32_t* next_out) {
    const NvtxRange nvtx(step == 0 ? "klotski step (prefill)" : "klotski step (decode)");
    if (cfg_.plan_only) throw ConfigError("engine: created with plan_only (no memory to run on)");
    if (step < 0 || step >= cfg_.workload.gen_len) throw RangeError("engine: step outside the batch group");
    if (step == 0 && !cfg_.prefill) throw ConfigError("engine: built without prefill support (prefill=false)");
    const int n = plan_.n_batches, bs = cfg_.workload.batch_size;
    const int tpb = tokens_per_batch(step);
    const int64_t T = static_cast<int64_t>(n) * tpb;
    // Host ids index the embedding table on the device: reject bad ones
    // before anything is enqueued (the caller provides exactly T of them).
    if (tokens_in != nullptr)
        for (int64_t i = 0; i < T; ++i)
            if (tokens_in[i] < 0 || tokens_in[i] >= D_.V)
                throw RangeError("engine: token id " + std::to_string(tokens_in[i]) + " outside the vocabulary");
    cur_step_ = step;
    executed_steps_.insert(step);
    const int64_t seqs = static_cast<int64_t>(n) * bs;
    cudaStream_t cs = stream_of(StreamId::compute);

    cudaEvent_t begin = event();
    cuda_check(cudaEventRecord(step_begin_, cs), "record");
    if (!t0_recorded_) kl_check(kl_stamp(stamps_dev_ + 2 * stamp_cap_, cs), "t0 stamp");
    cuda_check(cudaEventRecord(begin, cs), "record");
    for (int s = 1; s < kNumStreams; ++s) cuda_check(cudaStreamWaitEvent(streams_[s], begin, 0), "wait");

    // Token positions / cache rows; row order = batch-major, sequence-major.
    int32_t* hp = host_tokens_;
    int32_t* hs = host_tokens_ + t_max_;
    int32_t* hl = host_tokens_ + 2 * t_max_;
    int32_t* hsl = host_tokens_ + 4 * t_max_;
    for (int64_t r = 0; r < T; ++r) {
        const int64_t b = r / tpb, within = r % tpb;
        const int64_t sq = step == 0 ? within / cfg_.workload.prompt_len : within;
        hp[r] = step == 0 ? static_cast<int32_t>(within % cfg_.workload.prompt_len)
                          : cfg_.workload.prompt_len + step - 1;
        hs[r] = static_cast<int32_t>(b * bs + sq);
        hsl[r] = static_cast<int32_t>(sq);
    }
    if (kv_offload_)
        cuda_check(cudaMemcpyAsync(tok_seq_local_, hsl, T * 4, cudaMemcpyHostToDevice, cs), "h2d seq local");
    for (int64_t s = 0; s < seqs; ++s) {
        // Row of each sequence's last token this step (greedy head input).
        const int64_t b = s / bs, i = s % bs;
        hl[s] = static_cast<int32_t>(step == 0 ? b * tpb + i * cfg_.workload.prompt_len + cfg_.workload.prompt_len - 1
                                               : b * tpb + i);
    }
    cuda_check(cudaMemcpyAsync(tok_pos_, hp, T * 4, cudaMemcpyHostToDevice, cs), "h2d pos");
    cuda_check(cudaMemcpyAsync(tok_seq_, hs, T * 4, cudaMemcpyHostToDevice, cs), "h2d seq");
    cuda_check(cudaMemcpyAsync(last_rows_, hl, seqs * 4, cudaMemcpyHostToDevice, cs), "h2d rows");
    if (tokens_in != nullptr) {
        int32_t* ht = host_tokens_ + 3 * t_max_;
        std::memcpy(ht, tokens_in, T * 4);
        cuda_check(cudaMemcpyAsync(ids_, ht, T * 4, cudaMemcpyHostToDevice, cs), "h2d tokens");
    } else if (step == 0) {
        throw ConfigError("engine: prefill needs input tokens");
    } else {
        cuda_check(cudaMemcpyAsync(ids_, next_ids_, T * 4, cudaMemcpyDeviceToDevice, cs), "d2d tokens");
    }
    kl_check(kl_embed(ids_, embed_, T, D_.d, h_, cs), "embed");

    const bool split = em_->split_moe();
    if (cfg_.variant == Variant::simple) {
        // Row-by-row (schedule.cpp:636-690): each batch traverses every layer
        // alone, reloading each block's weights; the host reads the routing
        // of every (batch, layer) row before emitting its expert computes.
        for (int b = 0; b < n; ++b)
            for (int layer = 0; layer < D_.L; ++layer) {
                if (cfg_.replay) {
                    const auto sel = replay_trace_.layer_selections(step, layer);
                    for (size_t i = 0; i < sel.size(); ++i) host_forced_[i] = sel[i];
                }
                const detail::SimpleRow row = em_->simple_open(step, b, layer);
                block_layer_ = layer;
                issue_pending();
                const detail::BlockRouting routing = read_routing_row(step, layer, b);
                const std::int32_t first = static_cast<std::int32_t>(em_->schedule().ops.size());
                em_->simple_close(row, routing);
                block_defer_ = 0;
                exec_expert_left_ = 0;
                for (std::int32_t id = first; id < static_cast<std::int32_t>(em_->schedule().ops.size()); ++id)
                    exec_expert_left_ += em_->schedule().ops[id].kind == OpKind::compute_expert;
                issue_pending();
            }
    }
    for (int layer = 0; layer < D_.L && cfg_.variant != Variant::simple; ++layer) {
        PrefetchDecision d;
        if (!ep_) take_scores();  // the previous block's scores (its gate op has long been enqueued)
        if (split) d = decide(step, layer);
        if (cfg_.replay) {
            // Forced routing of this (step, layer) from the replay trace.
            const auto sel = replay_trace_.layer_selections(step, layer);
            for (size_t i = 0; i < sel.size(); ++i) host_forced_[i] = sel[i];
        }
        detail::OpenBlock blk = em_->open_block(step, layer, split ? &d : nullptr);
        block_layer_ = layer;
        issue_pending();
        const detail::BlockRouting routing = ep_ ? ep_read_routing(step, layer) : read_routing(step, layer);
        const detail::ClosedBlock closed = em_->close_block(blk, routing);
        exec_expert_left_ = 0;
        for (std::int32_t id = closed.first_op; id < static_cast<std::int32_t>(em_->schedule().ops.size()); ++id)
            exec_expert_left_ += em_->schedule().ops[id].kind == OpKind::compute_expert;
        block_defer_ = block_defer_splits(closed.first_op);
        if (ep_) ep_dispatch();  // routed rows to their expert's rank (every rank, every layer)
        issue_pending();
        if (ep_) ep_return(T);   // expert outputs back + weighted combine
    }

    // Greedy head on the last token of every sequence.
    kl_check(kl_embed(last_rows_, h_, seqs, D_.d, last_h_, cs), "gather last rows");
    kl_check(kl_rmsnorm(last_h_, final_norm_, seqs, D_.d, D_.eps, x2_, cs), "final norm");
    kl_check(kl_gemm_bf16(x2_, seqs, 0, static_cast<int>(seqs), D_.d, head_, D_.V, head_logits_, D_.V, nullptr, 0, gemm_ws_, gemm_ws_bytes_, cs),
             "lm head");
    kl_check(kl_argmax_bf16(head_logits_, seqs, D_.V, next_ids_, cs), "argmax");
    if (next_out != nullptr) {
        int32_t* ho = host_tokens_ + 3 * t_max_;
        cuda_check(cudaMemcpyAsync(ho, next_ids_, seqs * 4, cudaMemcpyDeviceToHost, cs), "d2h next");
    }
    // Join every stream into the end marker.
    for (int s = 1; s < kNumStreams; ++s) {
        cudaEvent_t j = event();
        cuda_check(cudaEventRecord(j, streams_[s]), "record");
        cuda_check(cudaStreamWaitEvent(cs, j, 0), "wait");
    }
    cuda_check(cudaEventRecord(step_end_, cs), "record");
    cuda_check(cudaEventSynchronize(step_end_), "step sync");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, step_begin_, step_end_), "elapsed");
    if (next_out != nullptr) std::memcpy(next_out, host_tokens_ + 3 * t_max_, seqs * 4);
    collect_step_times();
    tokens_generated_ += seqs;
    step_ms_.push_back(ms);
    return ms;
}

// End of a synchronized step: read back this step's op timestamps (one small
// D2H), turn them into timeline entries, and recycle the step's events and
// slot release markers.
void Engine::collect_step_times() {
    const auto& ops = em_->schedule().ops;
    const std::int64_t n_ops = next_exec_ - timed_from_;
    if (!t0_recorded_) {
        cuda_check(cudaMemcpy(stamps_host_ + 2 * stamp_cap_, stamps_dev_ + 2 * stamp_cap_, 8, cudaMemcpyDeviceToHost),
                   "d2h t0");
        t0_ns_ = stamps_host_[2 * stamp_cap_];
        t0_recorded_ = true;
    }
    if (n_ops > 0)
        cuda_check(cudaMemcpy(stamps_host_, stamps_dev_, static_cast<size_t>(n_ops) * 16, cudaMemcpyDeviceToHost),
                   "d2h stamps");
    if (timeline_.size() < ops.size()) timeline_.resize(ops.size());
    auto ps = [&](unsigned long long ns) {
        return static_cast<duration_ps>(static_cast<long long>(ns - t0_ns_)) * 1000;
    };
    for (std::int32_t id = timed_from_; id < next_exec_; ++id) {
        const unsigned long long* t = stamps_host_ + 2 * (id - timed_from_);
        SimEvent& ev = timeline_[id];
        ev.op_id = id;
        ev.stream = ops[id].stream;
        ev.start = ps(t[0]);
        ev.end = std::max(ev.start, ps(t[1]));
        ev.bytes = ops[id].payload_bytes;
        ev.tokens = ops[id].token_count;
    }
    timed_from_ = next_exec_;
    event_par_ ^= 1;
    event_next_ = 0;
    // Everything this step enqueued has completed: release markers can be
    // recycled.
    std::fill(pool_.has_release.begin(), pool_.has_release.end(), 0);
    std::fill(attn_slot_release_.begin(), attn_slot_release_.end(), nullptr);
    std::fill(gate_slot_release_.begin(), gate_slot_release_.end(), nullptr);
    std::fill(kv_slot_release_.begin(), kv_slot_release_.end(), nullptr);
    if (!kv_slot_of_.empty()) throw AccountingError("engine: KV slot still mapped at the end of a step");
    stage_jobs_.clear();
    if (const int e = stage_errno_.exchange(0))
        throw moesim::DeviceError(std::string("engine: disk staging read failed: ") + std::strerror(e));
}

// Enqueue every emitted-but-not-executed op. Cold computes of a reorder
// group on a VRAM-resident layer run in ascending expert id (they are all
// ready at the last gate, the simulator's tie rule, simulator.cpp:167-183);
// on streamed layers the FIFO expert_load stream completes colds in demand
// order, which is the simulator's earliest-ready pick.
void Engine::issue_pending() {
    const auto& ops = em_->schedule().ops;
    const std::int32_t total = static_cast<std::int32_t>(ops.size());
    if (static_cast<std::int32_t>(op_end_.size()) < total) op_end_.resize(total, nullptr);
    while (next_exec_ < total) {
        const StreamOp& op = ops[next_exec_];
        if (op.kind == OpKind::compute_expert && op.reorder_group >= 0 &&
            plan_.placement.expert_tier[op.layer] == Tier::vram) {
            std::int32_t end = next_exec_;
            while (end < total && ops[end].reorder_group == op.reorder_group) ++end;
            std::vector<std::int32_t> group(end - next_exec_);
            std::iota(group.begin(), group.end(), next_exec_);
            std::stable_sort(group.begin(), group.end(),
                             [&](std::int32_t a, std::int32_t b) { return ops[a].expert < ops[b].expert; });
            for (std::int32_t id : group) exec(id);
            next_exec_ = end;
            continue;
        }
        exec(next_exec_);
        ++next_exec_;
    }
}

// A dependency whose event has already completed needs no stream wait; a
// skipped wait keeps the stream's programmatic-dependent-launch chain intact
// (a cudaStreamWaitEvent between two kernels makes the second one wait for
// the first to finish before it can launch).
static void wait_unless_done(cudaStream_t st, cudaEvent_t ev, const char* what) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) cuda_check(q, what);
    cuda_check(cudaStreamWaitEvent(st, ev, 0), what);
}

void Engine::exec(std::int32_t id) {
    const StreamOp& op = em_->schedule().ops[id];
    const NvtxRange nvtx(op_kind_name(op.kind));
    cudaStream_t st = stream_of(op.stream);
    for (std::int32_t d : op.deps) {
        if (d < timed_from_) continue;  // finished in an earlier (synchronized) step
        if (em_->schedule().ops[d].stream == op.stream) continue;  // FIFO on the same stream
        wait_unless_done(st, op_end_[d], "dep wait");
    }
    op_end_[id] = event();
    cur_op_ = id;
    end_set_ = false;
    const size_t E = static_cast<size_t>(El_);  // local expert shard
    auto wait_release = [&](cudaEvent_t ev) {
        if (ev != nullptr) wait_unless_done(st, ev, "slot wait");
    };
    auto pick2 = [](std::vector<int>& busy) {
        for (int i = 0; i < 2; ++i)
            if (!busy[i]) {
                busy[i] = 1;
                return i;
            }
        throw AccountingError("engine: weight slot pool (2) exhausted");
    };

    switch (op.kind) {
        case OpKind::load_weights: {
            // Backpressure first (a slot may still be read by its previous user).
            if (op.cls == TensorClass::attention) {
                const int s = pick2(attn_slot_busy_);
                wait_release(attn_slot_release_[s]);
                stamp(id, 0, st);
                cuda_check(cudaMemcpyAsync(attn_slot_[s], load_src(TensorClass::attention, op.layer, 0, st), attn_slot_bytes_,
                                           cudaMemcpyHostToDevice, st), "h2d attention");
                attn_slot_of_[op.layer] = s;
            } else if (op.cls == TensorClass::gate) {
                const int s = pick2(gate_slot_busy_);
                wait_release(gate_slot_release_[s]);
                stamp(id, 0, st);
                cuda_check(cudaMemcpyAsync(gate_slot_[s], load_src(TensorClass::gate, op.layer, 0, st), spec_.gate_bytes,
                                           cudaMemcpyHostToDevice, st), "h2d gate");
                gate_slot_of_[op.layer] = s;
            } else {
                // Whole MoE layer (baseline variants): gate + every expert.
                const int s = pick2(gate_slot_busy_);
                wait_release(gate_slot_release_[s]);
                std::vector<int> slots;
                for (size_t e = 0; e < E; ++e) {
                    const int x = pool_.acquire();
                    if (pool_.has_release[x]) wait_release(pool_.release[x]);
                    slots.push_back(x);
                }
                stamp(id, 0, st);
                cuda_check(cudaMemcpyAsync(gate_slot_[s], load_src(TensorClass::gate, op.layer, 0, st), spec_.gate_bytes,
                                           cudaMemcpyHostToDevice, st), "h2d gate");
                for (size_t e = 0; e < E; ++e) {
                    cuda_check(cudaMemcpyAsync(pool_.ptr[slots[e]], load_src(TensorClass::expert, op.layer, static_cast<int>(e), st), expert_slot_bytes_,
                                               cudaMemcpyHostToDevice, st), "h2d moe");
                    expert_slot_of_[{op.layer, static_cast<int>(e)}] = slots[e];
                }
                gate_slot_of_[op.layer] = s;
                moe_slots_of_[op.layer] = slots;
            }
            break;
        }
        case OpKind::load_expert: {
            const int s = pool_.acquire();
            if (pool_.has_release[s]) wait_release(pool_.release[s]);
            stamp(id, 0, st);
            cuda_check(cudaMemcpyAsync(pool_.ptr[s], load_src(TensorClass::expert, op.layer, op.expert, st), expert_slot_bytes_,
                                       cudaMemcpyHostToDevice, st), "h2d expert");
            expert_slot_of_[{op.layer, op.expert}] = s;
            break;
        }
        case OpKind::offload_expert: {
            stamp(id, 0, st);
            const auto it = expert_slot_of_.find({op.layer, op.expert});
            if (it == expert_slot_of_.end()) throw AccountingError("engine: offload of an unloaded expert");
            // The slot is free once the offload op itself has completed (the
            // ledger frees at the offload's end), not merely its compute dep.
            pool_.release_after(it->second, op_end_[id]);
            expert_slot_of_.erase(it);
            break;
        }
        case OpKind::offload_weights: {
            stamp(id, 0, st);
            cudaEvent_t after = op_end_[id];  // recorded after the dep wait above
            if (op.cls == TensorClass::attention) {
                const int s = attn_slot_of_.at(op.layer);
                attn_slot_busy_[s] = 0;
                attn_slot_release_[s] = after;
                attn_slot_of_.erase(op.layer);
            } else {
                const int s = gate_slot_of_.at(op.layer);
                gate_slot_busy_[s] = 0;
                gate_slot_release_[s] = after;
                gate_slot_of_.erase(op.layer);
                const auto m = moe_slots_of_.find(op.layer);
                if (m != moe_slots_of_.end()) {
                    for (size_t e = 0; e < m->second.size(); ++e) {
                        pool_.release_after(m->second[e], after);
                        expert_slot_of_.erase({op.layer, static_cast<int>(e)});
                    }
                    moe_slots_of_.erase(m);
                }
            }
            break;
        }
        case OpKind::load_cache: {
            // Retained KV history of one (layer, batch) from pinned host into a
            // free device slot (load_kv, schedule.cpp:255-268): rows
            // [0, history) of every sequence, one 2D copy each for K and V.
            const int slot = acquire_kv_slot(st);
            stamp(id, 0, st);
            const int history = plan_.placement.kv_retention.retained(cfg_.workload.prompt_len + op.step - 1);
            const size_t row = static_cast<size_t>(D_.Hkv) * D_.hd * 2, pitch = row * kv_cap_;
            const uint16_t* h = host_kv_[static_cast<size_t>(op.layer) * plan_.n_batches + op.batch];
            const size_t half = kv_slot_bytes_ / 4;  // elements of K
            cuda_check(cudaMemcpy2DAsync(kv_slot_k_[slot], pitch, h, pitch, row * history, cfg_.workload.batch_size,
                                         cudaMemcpyHostToDevice, st), "h2d kv");
            cuda_check(cudaMemcpy2DAsync(kv_slot_v_[slot], pitch, h + half, pitch, row * history,
                                         cfg_.workload.batch_size, cudaMemcpyHostToDevice, st), "h2d kv");
            kv_slot_of_[{op.layer, op.batch}] = slot;
            break;
        }
        case OpKind::store_cache: {
            // This step's new K/V rows back to host (store_kv, schedule.cpp:270-288);
            // the slot is free once the copy has read it.
            stamp(id, 0, st);
            const auto it = kv_slot_of_.find({op.layer, op.batch});
            if (it == kv_slot_of_.end()) throw AccountingError("engine: KV store without a device slot");
            const int slot = it->second;
            const size_t row = static_cast<size_t>(D_.Hkv) * D_.hd * 2, pitch = row * kv_cap_;
            uint16_t* h = host_kv_[static_cast<size_t>(op.layer) * plan_.n_batches + op.batch];
            const size_t half = kv_slot_bytes_ / 4;
            size_t first = 0, rows = 0;
            if (op.step == 0) {
                rows = static_cast<size_t>(std::min(cfg_.workload.prompt_len, kv_cap_));
            } else {
                const int p = cfg_.workload.prompt_len + op.step - 1;
                first = static_cast<size_t>(p < kv_sink_ ? p : kv_sink_ + (p - kv_sink_) % (kv_cap_ - kv_sink_));
                rows = 1;
            }
            const size_t off = first * row / 2;
            cuda_check(cudaMemcpy2DAsync(h + off, pitch, kv_slot_k_[slot] + off, pitch, row * rows,
                                         cfg_.workload.batch_size, cudaMemcpyDeviceToHost, st), "d2h kv");
            cuda_check(cudaMemcpy2DAsync(h + half + off, pitch, kv_slot_v_[slot] + off, pitch, row * rows,
                                         cfg_.workload.batch_size, cudaMemcpyDeviceToHost, st), "d2h kv");
            kv_slot_release_[slot] = op_end_[id];
            kv_slot_of_.erase(it);
            break;
        }
        case OpKind::window_stage: {
            // Evict op.batch's window slot (its loads of this pass are the
            // op's deps), then read the staged layer's disk region into a
            // free slot on the cpu_stage stream (schedule.cpp:374-426).
            stamp(id, 0, st);
            const int evict = op.batch;
            if (evict >= 0 && window_slot_of_[evict] >= 0) {
                window_free_.push_back(window_slot_of_[evict]);
                window_slot_of_[evict] = -1;
            }
            if (disk_bytes(op.layer) > 0) {
                if (window_free_.empty()) throw AccountingError("engine: DRAM staging window has no free slot");
                if (window_slot_of_[op.layer] >= 0) throw AccountingError("engine: layer staged twice");
                const int slot = window_free_.front();
                window_free_.pop_front();
                window_slot_of_[op.layer] = slot;
                enqueue_disk_read(window_slot_[slot], disk_off_[op.layer], disk_bytes(op.layer), st);
            }
            break;
        }
        case OpKind::compute_attention:
            // bf16 decode: the op's first kernel (row RMSNorm) marks its start.
            if (op.step != 0 && !cfg_.quant)
                start_mark_ = id;
            else
                stamp(id, 0, st);
            exec_attention(op);
            if (start_mark_ >= 0) throw AccountingError("engine: attention op start mark not taken");
            break;
        case OpKind::compute_gate:
            // The router kernel marks the start when it is the op's first launch.
            if (cfg_.variant != Variant::simple && !cfg_.replay && op.batch != 0)
                start_mark_ = id;
            else
                stamp(id, 0, st);
            exec_gate(op);
            if (start_mark_ >= 0) throw AccountingError("engine: gate op start mark not taken");
            break;
        case OpKind::compute_expert:
            // bf16 experts: the op's first GEMM marks its start itself.
            if (op.token_count > 0 && !cfg_.quant)
                stamp_next_launch(id);
            else
                stamp(id, 0, st);
            exec_expert(op);
            break;
        default:
            throw ConfigError(std::string("engine: op kind ") + op_kind_name(op.kind) + " is not executed on B200 yet");
    }
    if (combine_step_ >= 0) {
        // The block's weighted combine (and, with deferred splits, the
        // down-projection reduction it carries) belongs to its last expert op.
        combine_block(combine_step_);
        combine_step_ = -1;
    }
    if (!end_set_ || kl_stamp_end_pending()) stamp(id, 1, st);
    end_set_ = false;
    cuda_check(cudaEventRecord(op_end_[id], st), "record");
}

void Engine::exec_attention(const StreamOp& op) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int l = op.layer, step = op.step, b = op.batch;
    const int tpb = tokens_per_batch(step);
    const int64_t row0 = static_cast<int64_t>(b) * tpb;
    const uint16_t* w = res_attn_[l] ? res_attn_[l] : attn_slot_[attn_slot_of_.at(l)];
    // Streamed attention weights arrive as Q4T when quantised: fused-dequant
    // GEMMs for decode-sized batches, dequantise-then-bf16 for prefill.
    const bool q4 = cfg_.quant && res_attn_[l] == nullptr;
    const int64_t wo_k = static_cast<int64_t>(D_.Hq) * D_.hd;
    const uint8_t* q4qkv = reinterpret_cast<const uint8_t*>(w);
    const uint8_t* q4o = q4qkv + kl_q4_bytes(D_.qkv_width(), D_.d);
    if (q4 && tpb > 256) {
        kl_check(kl_dequantize_q4(q4qkv, D_.qkv_width(), D_.d, wscratch_, cs), "dequant qkv");
        kl_check(kl_dequantize_q4(q4o, D_.d, wo_k, wscratch_ + static_cast<int64_t>(D_.qkv_width()) * D_.d, cs),
                 "dequant o");
        w = wscratch_;
    }
    const bool fused = q4 && tpb <= 256;
    const uint16_t* wqkv = w;
    const uint16_t* wo = w + static_cast<int64_t>(D_.qkv_width()) * D_.d;
    uint16_t* hb = h_ + row0 * D_.d;
    const float scale = 1.0f / std::sqrt(static_cast<float>(D_.hd));
    const int last = step == 0 ? cfg_.workload.prompt_len - 1 : -1;
    uint16_t* kc = kc_[l];
    uint16_t* vc = vc_[l];
    const int32_t* seq_idx = tok_seq_ + row0;
    if (kv_offload_) {
        // The batch's KV slot (loaded by load_cache; a fresh one for prefill).
        auto it = kv_slot_of_.find({l, b});
        if (it == kv_slot_of_.end()) {
            if (step != 0) throw AccountingError("engine: decode attention without a loaded KV slot");
            it = kv_slot_of_.emplace(std::make_pair(l, b), acquire_kv_slot(cs)).first;
        }
        kc = kv_slot_k_[it->second];
        vc = kv_slot_v_[it->second];
        seq_idx = tok_seq_local_ + row0;
    }
    // Decode with bf16 projections, opt-in (KL_QKV_ROPE=1): RMSNorm writes the
    // RoPE table and the QKV GEMM rotates q / k and appends k / v in its
    // epilogue (two launches instead of three); shapes off the weight-
    // streaming path fall back.
    if (step != 0 && !fused && rope_fused_ok_) {
        take_start_mark();
        kl_check(kl_rmsnorm_rope_table(hb, norm_attn_[l], tpb, D_.d, D_.eps, xa_, tok_pos_ + row0, D_.theta, D_.hd,
                                       rope_tab_, cs), "attn norm + rope table");
        const int rc = kl_gemm_bf16_qkv_rope(xa_, tpb, 0, tpb, D_.d, wqkv, D_.Hq, D_.Hkv, D_.hd, qkv_, D_.qkv_width(),
                                             rope_tab_, tok_pos_ + row0, seq_idx, kc, vc, kv_cap_, kv_sink_, -1,
                                             gemm_ws_, gemm_ws_bytes_, cs);
        if (rc == KL_EUNSUPPORTED) {
            rope_fused_ok_ = false;  // this engine's shapes take the separate calls from now on
            kl_check(kl_gemm_bf16(xa_, tpb, 0, tpb, D_.d, wqkv, D_.qkv_width(), qkv_, D_.qkv_width(), nullptr, 0,
                                  gemm_ws_, gemm_ws_bytes_, cs), "qkv");
            kl_check(kl_rope_kv_append(qkv_, tpb, D_.Hq, D_.Hkv, D_.hd, tok_pos_ + row0, seq_idx, D_.theta, kc, vc,
                                       kv_cap_, kv_sink_, last, cs), "rope/kv");
        } else {
            kl_check(rc, "qkv + rope/kv");
        }
    } else if (step != 0 && !fused && defer_ok_ && qkvpart_ != nullptr &&
               (qkv_defer_ < 0 ? (qkv_defer_ = kl_gemm_deferred_splits(tpb, D_.qkv_width(), D_.d)) : qkv_defer_) > 0) {
        // Decode: the QKV GEMM leaves its tile-aligned k-splits as fp32
        // partials and the RoPE / KV-append kernel sums them (no fixup tail).
        take_start_mark();
        kl_check(kl_rmsnorm(hb, norm_attn_[l], tpb, D_.d, D_.eps, xa_, cs), "attn norm");
        kl_check(kl_gemm_bf16_deferred(xa_, tpb, 0, tpb, D_.d, wqkv, D_.qkv_width(), 0, qkvpart_,
                                       cfg_.workload.batch_size, qkv_defer_, gemm_ws_, gemm_ws_bytes_, cs),
                 "qkv (deferred splits)");
        kl_check(kl_rope_kv_append_deferred(qkvpart_, qkv_defer_, cfg_.workload.batch_size, qkv_, tpb, D_.Hq, D_.Hkv,
                                            D_.hd, tok_pos_ + row0, seq_idx, D_.theta, kc, vc, kv_cap_, kv_sink_, -1,
                                            cs),
                 "rope/kv (deferred splits)");
    } else {
        take_start_mark();
        kl_check(kl_rmsnorm(hb, norm_attn_[l], tpb, D_.d, D_.eps, xa_, cs), "attn norm");
        if (fused)
            kl_check(kl_gemm_q4(xa_, tpb, 0, tpb, D_.d, q4qkv, D_.qkv_width(), qkv_, D_.qkv_width(), nullptr, 0, gemm_ws_,
                                gemm_ws_bytes_, cs), "qkv q4");
        else
            kl_check(kl_gemm_bf16(xa_, tpb, 0, tpb, D_.d, wqkv, D_.qkv_width(), qkv_, D_.qkv_width(), nullptr, 0,
                                  gemm_ws_, gemm_ws_bytes_, cs), "qkv");
        kl_check(kl_rope_kv_append(qkv_, tpb, D_.Hq, D_.Hkv, D_.hd, tok_pos_ + row0, seq_idx, D_.theta, kc, vc, kv_cap_,
                                   kv_sink_, last, cs), "rope/kv");
    }
    if (step == 0)
        kl_check(kl_attn_prefill(qkv_, cfg_.workload.batch_size, cfg_.workload.prompt_len, D_.Hq, D_.Hkv, D_.hd,
                                 kv_cap_, kv_sink_, scale, ao_, cs), "prefill attention");
    else
        kl_check(kl_attn_decode_ws2(qkv_, D_.qkv_width(), tok_pos_ + row0, seq_idx, tpb, D_.Hq, D_.Hkv, D_.hd, kc, vc,
                                    static_cast<int64_t>(cfg_.workload.batch_size) * (kv_offload_ ? 1 : plan_.n_batches),
                                    kv_cap_, kv_sink_, scale, ao_, gemm_ws_, gemm_ws_bytes_, cs),
                 "decode attention");
    const int64_t wo_k2 = static_cast<int64_t>(D_.Hq) * D_.hd;
    if (fused) {
        kl_check(kl_gemm_q4(ao_, tpb, 0, tpb, D_.Hq * D_.hd, q4o, D_.d, hb, D_.d, hb, 1, gemm_ws_, gemm_ws_bytes_, cs),
                 "o proj q4");
    } else if (step != 0 && defer_ok_ && opart_ != nullptr && tpb <= 4 * 148 && D_.d % 256 == 0 &&
               (D_.d / 256 == 2 || D_.d / 256 == 4 || D_.d / 256 == 8 || D_.d / 256 == 16 || D_.d / 256 == 24) &&
               (o_defer_ < 0 ? (o_defer_ = kl_gemm_deferred_splits(tpb, D_.d, static_cast<int>(wo_k2))) : o_defer_) > 0) {
        // Decode: the o-proj leaves its tile-aligned k-splits as fp32 partials;
        // this batch's gate op completes h (+ residual) before its router.
        end_mark_next();  // the op's last launch
        kl_check(kl_gemm_bf16_deferred(ao_, tpb, 0, tpb, static_cast<int>(wo_k2), wo, D_.d, 0,
                                       opart_ + static_cast<int64_t>(b) * 4 * cfg_.workload.batch_size * D_.d,
                                       cfg_.workload.batch_size, o_defer_, gemm_ws_, gemm_ws_bytes_, cs),
                 "o proj (deferred splits)");
        o_deferred_[static_cast<size_t>(b)] = o_defer_;
    } else {
        kl_check(kl_gemm_bf16(ao_, tpb, 0, tpb, D_.Hq * D_.hd, wo, D_.d, hb, D_.d, hb, 1, gemm_ws_, gemm_ws_bytes_, cs),
                 "o proj");
    }
}

void Engine::exec_gate(const StreamOp& op) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int l = op.layer, step = op.step, b = op.batch;
    const int n = plan_.n_batches;
    const int tpb = tokens_per_batch(step);
    const int64_t row0 = static_cast<int64_t>(b) * tpb;
    int32_t* hist = report_ + static_cast<int64_t>(b) * D_.E;
    int32_t* first = report_ + static_cast<int64_t>(n) * D_.E + static_cast<int64_t>(b) * D_.E;
    const bool simple = cfg_.variant == Variant::simple;
    if (simple) {
        // One batch per row: clear only this batch's histogram / first demand.
        cuda_check(cudaMemsetAsync(hist, 0, static_cast<size_t>(D_.E) * 4, cs), "memset hist");
        cuda_check(cudaMemsetAsync(first, 0x7f, static_cast<size_t>(D_.E) * 4, cs), "memset first");
        if (cfg_.replay)
            cuda_check(cudaMemcpyAsync(forced_ + row0 * D_.k, host_forced_ + row0 * D_.k,
                                       static_cast<size_t>(tpb) * D_.k * 4, cudaMemcpyHostToDevice, cs),
                       "h2d forced routing");
    } else if (b == 0) {
        if (readback_pending_) {  // the previous block's readback copies have read the report
            cuda_check(cudaStreamWaitEvent(cs, scores_ready_, 0), "wait readback");
            readback_pending_ = false;
        }
        cuda_check(cudaMemsetAsync(report_, 0, static_cast<size_t>(n) * D_.E * 4, cs), "memset hist");
        cuda_check(cudaMemsetAsync(report_ + static_cast<int64_t>(n) * D_.E, 0x7f, static_cast<size_t>(n) * D_.E * 4, cs),
                   "memset first");
        if (cfg_.replay)
            cuda_check(cudaMemcpyAsync(forced_, host_forced_, static_cast<size_t>(n) * tpb * D_.k * 4,
                                       cudaMemcpyHostToDevice, cs), "h2d forced routing");
    }
    const uint16_t* wg = gate_slot_[gate_slot_of_.at(l)];
    int32_t* idx = idx_[idx_cur_] + row0 * D_.k;
    float* wt = weight_ + row0 * D_.k;
    const int odef = o_deferred_.empty() ? 0 : o_deferred_[static_cast<size_t>(b)];
    take_start_mark();
    if (!simple && !cfg_.replay && b != n - 1) end_mark_next();  // the router is the op's only launch
    if (odef > 0) {
        // This batch's o-proj left split partials: the router kernel completes h first.
        o_deferred_[static_cast<size_t>(b)] = 0;
        const float* part = opart_ + static_cast<int64_t>(b) * 4 * cfg_.workload.batch_size * D_.d;
        kl_check(kl_gate_topk_deferred(h_ + row0 * D_.d, part, odef, cfg_.workload.batch_size, norm_ffn_[l], wg, tpb,
                                       D_.d, D_.E, D_.k, D_.eps, D_.score_mode, x2_ + row0 * D_.d,
                                       cfg_.replay ? router_logits_ + row0 * D_.E : nullptr, idx, wt,
                                       cfg_.replay ? nullptr : hist, cfg_.replay ? nullptr : first, cs),
                 "gate (deferred o-proj)");
        if (cfg_.replay)
            kl_check(kl_route_override(forced_ + row0 * D_.k, router_logits_ + row0 * D_.E, tpb, D_.E, D_.k, idx, wt,
                                       hist, first, cs), "route override");
    } else if (cfg_.replay) {
        kl_check(kl_gate_topk(h_ + row0 * D_.d, norm_ffn_[l], wg, tpb, D_.d, D_.E, D_.k, D_.eps, D_.score_mode,
                              x2_ + row0 * D_.d, router_logits_ + row0 * D_.E, idx, wt, nullptr, nullptr, cs), "gate");
        kl_check(kl_route_override(forced_ + row0 * D_.k, router_logits_ + row0 * D_.E, tpb, D_.E, D_.k, idx, wt, hist,
                                   first, cs), "route override");
    } else {
        kl_check(kl_gate_topk(h_ + row0 * D_.d, norm_ffn_[l], wg, tpb, D_.d, D_.E, D_.k, D_.eps, D_.score_mode,
                              x2_ + row0 * D_.d, nullptr, idx, wt, hist, first, cs), "gate");
    }
    if (simple)
        after_batch_gate(step, l, b);
    else if (b == n - 1) {
        if (ep_)
            ep_after_gates(step, l);
        else
            after_layer_gates(step, l);
    }
}

// Work tied to the block's last gate: expert-major permutation of the whole
// group, the prefetcher's online table update and the next layer's scores,
// then one small D2H of everything the host needs to emit the rest.
void Engine::after_layer_gates(int step, int layer) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int n = plan_.n_batches;
    const int64_t T = static_cast<int64_t>(n) * tokens_per_batch(step);
    int32_t* cur = idx_[idx_cur_];
    int32_t* prev = idx_[idx_cur_ ^ 1];
    // Part 1 of the readback: what close_block needs (per-batch histogram and
    // first demand, recorded ids), ahead of the permutation.
    // Copied on rb_stream_ behind gates_done_: the compute stream goes on to
    // the permutation without waiting for the PCIe round trip.
    cuda_check(cudaEventRecord(gates_done_, cs), "gates done");
    cuda_check(cudaStreamWaitEvent(rb_stream_, gates_done_, 0), "wait gates");
    cuda_check(cudaMemcpyAsync(host_report_, report_, 2LL * n * D_.E * 4, cudaMemcpyDeviceToHost, rb_stream_),
               "d2h routing");
    if (cfg_.record_trace)
        cuda_check(cudaMemcpyAsync(host_idx_, cur, T * D_.k * 4, cudaMemcpyDeviceToHost, rb_stream_), "d2h idx");
    cuda_check(cudaEventRecord(routing_ready_, rb_stream_), "routing ready");
    kl_check(kl_permute(cur, T, D_.k, D_.E, x2_, D_.d, counts_, offsets_, pos_, row_token_, xp_, perm_ws_, cs),
             "permute");
    shared_experts(layer, T, 0);
    launches_ += kl_permute_launches(T * D_.k) - 1;  // rank (+ scan) + scatter kernels
    int64_t* scores = reinterpret_cast<int64_t*>(report_ + 2LL * n * D_.E + 16 - ((2LL * n * D_.E) % 16));
    int64_t* marg_copy = scores + D_.E;
    if (layer + 1 < D_.L) {
        kl_check(kl_coact_update(layer == 0 ? nullptr : prev, cur, T, D_.k, D_.E, layer, table_, marginal_, cs),
                 "coact update");
        kl_check(kl_predict_scores(counts_, table_, D_.E, layer + 1, scores, cs), "predict");
    }
    cuda_check(cudaMemcpyAsync(marg_copy, marginal_, D_.E * 8, cudaMemcpyDeviceToDevice, cs), "marginal");
    // Part 2: the next layer's prefetch scores and the marginal (take_scores).
    const size_t head = reinterpret_cast<char*>(scores) - reinterpret_cast<char*>(report_);
    cuda_check(cudaEventRecord(scores_done_, cs), "scores done");
    cuda_check(cudaStreamWaitEvent(rb_stream_, scores_done_, 0), "wait scores");
    cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(host_report_) + head, scores, 2LL * D_.E * 8,
                               cudaMemcpyDeviceToHost, rb_stream_), "d2h scores");
    cuda_check(cudaEventRecord(scores_ready_, rb_stream_), "scores ready");
    scores_pending_ = true;
    readback_pending_ = true;
    idx_cur_ ^= 1;  // this layer's ids become "prev" for the next layer
}

// The prefetcher's next-layer scores of the last closed block (readback part
// 2), once its gate op has completed; before the next block's decision.
void Engine::take_scores() {
    if (!scores_pending_) return;
    cuda_check(cudaEventSynchronize(scores_ready_), "scores sync");
    scores_pending_ = false;
    const int n = plan_.n_batches, E = D_.E;
    const int64_t* scores =
        reinterpret_cast<const int64_t*>(host_report_ + 2LL * n * E + 16 - ((2LL * n * E) % 16));
    host_scores_.assign(scores, scores + E);
    host_marginal_.assign(scores + E, scores + 2 * E);
}

// Shared experts (always active): h += FFN_shared(x2) on every token of the
// group, from the router tensor's slot ([router E x d | W13s (2 fs x d) |
// W2s (d x fs)]); the combine then adds the routed experts on top.
void Engine::shared_experts(int layer, int64_t T, int64_t row0) {
    if (D_.fs() <= 0) return;
    cudaStream_t cs = stream_of(StreamId::compute);
    const uint16_t* g = gate_slot_[gate_slot_of_.at(layer)];
    const uint16_t* w13 = g + static_cast<int64_t>(D_.E) * D_.d;
    const uint16_t* w2 = w13 + 2LL * D_.fs() * D_.d;
    for (int64_t c = 0; c < T; c += cfg_.ffn_chunk_rows) {
        const int m = static_cast<int>(std::min<int64_t>(cfg_.ffn_chunk_rows, T - c));
        uint16_t* hrow = h_ + (row0 + c) * D_.d;
        kl_check(kl_gemm_bf16(x2_, row0 + T, row0 + c, m, D_.d, w13, 2 * D_.fs(), hshared_, D_.fs(), nullptr, 2,
                              gemm_ws_, gemm_ws_bytes_, cs), "shared w13");
        kl_check(kl_gemm_bf16(hshared_, m, 0, m, D_.fs(), w2, D_.d, hrow, D_.d, hrow, 1, gemm_ws_, gemm_ws_bytes_, cs),
                 "shared w2");
    }
}

// simple variant: the gate of ONE batch row is followed by that batch's own
// expert-major permutation (and shared experts) and a readback of its
// histogram / first demand (the reference's build_simple, schedule.cpp:636-690,
// routes each batch alone).
void Engine::after_batch_gate(int step, int layer, int b) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int tpb = tokens_per_batch(step);
    const int64_t row0 = static_cast<int64_t>(b) * tpb;
    int32_t* cur = idx_[idx_cur_] + row0 * D_.k;
    kl_check(kl_permute(cur, tpb, D_.k, D_.E, x2_ + row0 * D_.d, D_.d, counts_, offsets_, pos_ + row0 * D_.k,
                        row_token_ + row0 * D_.k, xp_, perm_ws_, cs), "permute (row)");
    launches_ += kl_permute_launches(static_cast<int64_t>(tpb) * D_.k) - 1;
    shared_experts(layer, tpb, row0);
    const int n = plan_.n_batches;
    const size_t hist_off = static_cast<size_t>(b) * D_.E, first_off = static_cast<size_t>(n) * D_.E + hist_off;
    cuda_check(cudaMemcpyAsync(host_report_ + hist_off, report_ + hist_off, D_.E * 4, cudaMemcpyDeviceToHost, cs),
               "d2h row hist");
    cuda_check(cudaMemcpyAsync(host_report_ + first_off, report_ + first_off, D_.E * 4, cudaMemcpyDeviceToHost, cs),
               "d2h row first");
    if (cfg_.record_trace)
        cuda_check(cudaMemcpyAsync(host_idx_ + row0 * D_.k, cur, static_cast<size_t>(tpb) * D_.k * 4,
                                   cudaMemcpyDeviceToHost, cs), "d2h row idx");
    (void)step;
}

detail::BlockRouting Engine::read_routing_row(int step, int layer, int b) {
    // The row's gate op (the last op issued) ends after its readback copies.
    cuda_check(cudaEventSynchronize(op_end_[next_exec_ - 1]), "routing sync");
    const int n = plan_.n_batches, E = D_.E;
    detail::BlockRouting r;
    r.group_hist.assign(E, 0);
    r.demand.resize(n);
    r.batch_hist.assign(n, std::vector<int64_t>(E, 0));
    std::vector<std::pair<int32_t, int>> firsts;
    for (int e = 0; e < E; ++e) {
        const int32_t c = host_report_[b * E + e];
        r.batch_hist[b][e] = c;
        r.group_hist[e] = c;
        if (c > 0) {
            const int32_t f = host_report_[n * E + b * E + e];
            if (f == kNoPos) throw AccountingError("engine: routed expert without a first position");
            firsts.emplace_back(f, e);
        }
    }
    std::sort(firsts.begin(), firsts.end());
    for (const auto& [f, e] : firsts) r.demand[b].push_back(e);
    // The row's permuted rows start at 0 in xp_ (this batch only).
    row_offset_.assign(E, 0);
    for (int e = 1; e < E; ++e) row_offset_[e] = row_offset_[e - 1] + r.group_hist[e - 1];
    block_rows_ = std::accumulate(r.group_hist.begin(), r.group_hist.end(), int64_t{0});
    batch_prefix_.assign(n, std::vector<int64_t>(E, 0));
    if (cfg_.record_trace) {
        const int tpb = tokens_per_batch(step);
        const size_t off = recorded_.offset(step, layer, b, 0);
        const int64_t row0 = static_cast<int64_t>(b) * tpb;
        for (int64_t i = 0; i < static_cast<int64_t>(tpb) * D_.k; ++i)
            recorded_.sel[off + i] = static_cast<uint16_t>(host_idx_[row0 * D_.k + i]);
    }
    return r;
}

detail::BlockRouting Engine::read_routing(int step, int layer) {
    // The last op issued on the compute stream is the block's last gate;
    // its end event covers the readback copies.
    cuda_check(cudaEventSynchronize(routing_ready_), "routing sync");
    const int n = plan_.n_batches, E = D_.E;
    detail::BlockRouting r;
    r.group_hist.assign(E, 0);
    r.demand.resize(n);
    r.batch_hist.assign(n, std::vector<int64_t>(E, 0));
    for (int b = 0; b < n; ++b) {
        std::vector<std::pair<int32_t, int>> firsts;
        for (int e = 0; e < E; ++e) {
            const int32_t c = host_report_[b * E + e];
            r.batch_hist[b][e] = c;
            r.group_hist[e] += c;
            const int32_t f = host_report_[n * E + b * E + e];
            if (c > 0) {
                if (f == kNoPos) throw AccountingError("engine: routed expert without a first position");
                firsts.emplace_back(f, e);
            }
        }
        std::sort(firsts.begin(), firsts.end());
        for (const auto& [f, e] : firsts) r.demand[b].push_back(e);
    }
    // Expert segment starts of the stable counting sort (== device offsets).
    row_offset_.assign(E, 0);
    for (int e = 1; e < E; ++e) row_offset_[e] = row_offset_[e - 1] + r.group_hist[e - 1];
    block_rows_ = std::accumulate(r.group_hist.begin(), r.group_hist.end(), int64_t{0});
    batch_prefix_.assign(n, std::vector<int64_t>(E, 0));
    for (int b = 1; b < n; ++b)
        for (int e = 0; e < E; ++e) batch_prefix_[b][e] = batch_prefix_[b - 1][e] + r.batch_hist[b - 1][e];
    if (cfg_.record_trace) {
        const size_t off = recorded_.offset(step, layer, 0, 0);
        const int64_t cnt = static_cast<int64_t>(n) * tokens_per_batch(step) * D_.k;
        for (int64_t i = 0; i < cnt; ++i) recorded_.sel[off + i] = static_cast<uint16_t>(host_idx_[i]);
    }
    return r;
}

// Split count shared by every expert FFN of the block just closed when all of
// them can leave their down-projection splits for the combine (decode-sized
// rows, one chunk each, the same tile-aligned split); 0 otherwise.
int Engine::block_defer_splits(std::int32_t first_op) const {
    if (!defer_ok_ || ypart_ == nullptr || block_rows_ > ypart_rows_) return 0;
    const auto& ops = em_->schedule().ops;
    int S = -1;
    for (std::int32_t id = first_op; id < static_cast<std::int32_t>(ops.size()); ++id) {
        const StreamOp& o = ops[id];
        if (o.kind != OpKind::compute_expert || o.token_count == 0) continue;
        if (o.token_count > cfg_.ffn_chunk_rows) return 0;
        const int s = kl_expert_ffn_deferred_splits(static_cast<int>(o.token_count), D_.d, D_.f);
        if (s < 2 || (S >= 0 && s != S)) return 0;
        S = s;
    }
    return S > 0 ? S : 0;
}

void Engine::exec_expert(const StreamOp& op) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int l = op.layer, e = op.expert;
    const int64_t M = op.token_count;
    const int64_t row0 = row_offset_[e] + (op.batch >= 0 ? batch_prefix_[op.batch][e] : 0);  // simple: prefix 0
    const uint16_t* w = expert_weights(l, e);
    const bool q4 = cfg_.quant && res_expert_[static_cast<size_t>(l) * El_ + e] == nullptr;
    const uint8_t* q13 = reinterpret_cast<const uint8_t*>(w);
    const uint8_t* q2 = q13 + kl_q4_bytes(2LL * D_.f, D_.d);
    if (q4 && M > 256) {  // prefill-sized: expand once, then the compute-bound bf16 GEMMs
        kl_check(kl_dequantize_q4(q13, 2LL * D_.f, D_.d, wscratch_, cs), "dequant w13");
        kl_check(kl_dequantize_q4(q2, D_.d, D_.f, wscratch_ + 2LL * D_.f * D_.d, cs), "dequant w2");
        w = wscratch_;
    }
    const uint16_t* w2 = w + 2LL * D_.f * D_.d;
    for (int64_t c = 0; c < M; c += cfg_.ffn_chunk_rows) {
        const int m = static_cast<int>(std::min<int64_t>(cfg_.ffn_chunk_rows, M - c));
        if (q4 && M <= 256)
            kl_check(kl_expert_ffn_q4(xp_, block_rows_, row0 + c, m, D_.d, D_.f, q13, q2, hs_, y_, gemm_ws_,
                                      gemm_ws_bytes_, cs), "expert ffn q4");
        else if (block_defer_ > 0) {  // down-projection splits left for the block's combine to sum
            // The down GEMM is the op's last launch unless the block's combine follows.
            if (c + m >= M && !ep_ && exec_expert_left_ > 1) end_mark_next();
            kl_check(kl_expert_ffn_kb_deferred(xp_, block_rows_, row0 + c, m, D_.d, D_.f, w, w2, hs_, ypart_,
                                               ypart_rows_, block_defer_, gemm_ws_, gemm_ws_bytes_, cs),
                     "expert ffn (deferred splits)");
        }
        else if (expert_kblocked())  // bf16 experts (resident or streamed) are stored K-blocked
            kl_check(kl_expert_ffn_kb(xp_, block_rows_, row0 + c, m, D_.d, D_.f, w, w2, hs_, y_, gemm_ws_,
                                      gemm_ws_bytes_, cs), "expert ffn");
        else
            kl_check(kl_expert_ffn(xp_, block_rows_, row0 + c, m, D_.d, D_.f, w, w2, hs_, y_, gemm_ws_,
                                   gemm_ws_bytes_, cs), "expert ffn");
        ++launches_;  // gate/up (SwiGLU) GEMM + down GEMM
    }
    // The block's last expert op also runs the combine (exec(), before the
    // op's end stamp).
    if (--exec_expert_left_ == 0 && !ep_) {
        combine_step_ = op.step;
        combine_batch_ = cfg_.variant == Variant::simple ? op.batch : -1;
    }
}

void Engine::combine_block(int step) {
    // Every routed row of the block is computed: weighted combine + residual.
    cudaStream_t cs = stream_of(StreamId::compute);
    if (combine_batch_ >= 0) {  // simple: one batch row
        const int tpb = tokens_per_batch(step);
        const int64_t row0 = static_cast<int64_t>(combine_batch_) * tpb;
        uint16_t* hb = h_ + row0 * D_.d;
        kl_check(kl_combine(y_, pos_ + row0 * D_.k, weight_ + row0 * D_.k, hb, tpb, D_.k, D_.d, hb, cs), "combine");
        combine_batch_ = -1;
        if (cfg_.record_hidden) {  // one dump per (batch, layer) row: that batch's rows only
            std::vector<uint16_t> dump(static_cast<size_t>(tpb) * D_.d);
            cuda_check(cudaMemcpyAsync(dump.data(), hb, dump.size() * 2, cudaMemcpyDeviceToHost, cs), "dump");
            cuda_check(cudaStreamSynchronize(cs), "dump sync");
            hidden_dumps_.push_back(std::move(dump));
        }
        return;
    }
    const int64_t T = static_cast<int64_t>(plan_.n_batches) * tokens_per_batch(step);
    if (block_defer_ > 0)
        kl_check(kl_combine_deferred(ypart_, block_defer_, ypart_rows_, pos_, weight_, h_, T, D_.k, D_.d, h_, cs),
                 "combine (deferred splits)");
    else
        kl_check(kl_combine(y_, pos_, weight_, h_, T, D_.k, D_.d, h_, cs), "combine");
    if (cfg_.record_hidden) {
        std::vector<uint16_t> dump(static_cast<size_t>(T) * D_.d);
        cuda_check(cudaMemcpyAsync(dump.data(), h_, dump.size() * 2, cudaMemcpyDeviceToHost, cs), "dump");
        cuda_check(cudaStreamSynchronize(cs), "dump sync");
        hidden_dumps_.push_back(std::move(dump));
    }
}

void Engine::read_hidden(uint16_t* host, int64_t n) const {
    if (cfg_.plan_only) throw ConfigError("engine: created with plan_only (no hidden states)");
    cuda_check(cudaDeviceSynchronize(), "sync");
    cuda_check(cudaMemcpy(host, h_, static_cast<size_t>(std::min<int64_t>(n, t_max_ * D_.d)) * 2,
                          cudaMemcpyDeviceToHost), "read hidden");
}

void Engine::reset_log() {
    if (cfg_.plan_only) return;
    // Keep the emitter (op ids keep growing); measurement restarts here.
    timed_from_ = next_exec_;
    log_from_ = next_exec_;
    records_from_ = em_->schedule().prefetch_records.size();
    t0_recorded_ = false;
    tokens_generated_ = 0;
    launches_ = 0;
    ep_max_local_rows_ = 0;
    step_ms_.clear();
    hidden_dumps_.clear();
}

std::string Engine::report(const std::string& what) {
    if (cfg_.plan_only) throw ConfigError("engine: created with plan_only (nothing executed to report)");
    const Schedule& s = em_->schedule();
    json j;
    std::vector<SimEvent> tl(timeline_.begin() + std::min<size_t>(log_from_, timeline_.size()),
                             timeline_.begin() + std::min<size_t>(next_exec_, timeline_.size()));
    if (what == "schedule") {
        j["text"] = s.to_text();
        j["n_ops"] = s.ops.size();
    } else if (what == "timeline_csv") {
        j["text"] = timeline_to_string(tl, s, TimelineFormat::csv);
    } else if (what == "timeline_json") {
        j["text"] = timeline_to_string(tl, s, TimelineFormat::trace_event_json);
    } else if (what == "metrics") {
        j = reference_metrics(s, records_from_, tl, arena_used_, tokens_generated_);
        // Host-link accounting: bytes moved by load ops and the time the
        // link had at least one load in flight (union of load intervals).
        const auto [h2d, link_busy] = link_usage(s, tl);
        const duration_ps makespan = j["makespan_ps"].get<duration_ps>();
        int64_t n_expert_loads = 0;
        duration_ps expert_busy = 0;
        std::map<int, duration_ps> kind_busy;
        for (const SimEvent& e : tl) {
            const StreamOp& op = s.ops[e.op_id];
            if (op.kind == OpKind::load_expert) {
                ++n_expert_loads;
                expert_busy += e.end - e.start;
            }
            if (op.stream == StreamId::compute) kind_busy[static_cast<int>(op.kind)] += e.end - e.start;
        }
        j["h2d_bytes"] = h2d;
        j["h2d_link_busy_ps"] = link_busy;
        j["h2d_gbs_busy"] = link_busy > 0 ? h2d / (link_busy * 1e-12) / 1e9 : 0.0;
        j["h2d_gbs_makespan"] = makespan > 0 ? h2d / (makespan * 1e-12) / 1e9 : 0.0;
        j["expert_loads"] = n_expert_loads;
        j["expert_load_busy_ps"] = expert_busy;
        {
            int64_t n_stage = 0, stage_bytes = 0;
            duration_ps stage_busy = 0;
            for (const SimEvent& e : tl)
                if (s.ops[e.op_id].kind == OpKind::window_stage) {
                    ++n_stage;
                    stage_bytes += e.bytes;
                    stage_busy += e.end - e.start;
                }
            j["window_stages"] = n_stage;
            j["disk_stage_bytes"] = stage_bytes;
            j["disk_bytes_read"] = disk_bytes_read_.load();
            j["disk_direct_reads"] = direct_reads_;
            j["disk_direct_bytes"] = direct_bytes_;
            j["disk_gbs_busy"] = stage_busy > 0 ? stage_bytes / (stage_busy * 1e-12) / 1e9 : 0.0;
        }
        j["launches"] = launches_;
        if (ep_) {
            j["ep_world"] = G_;
            j["ep_rank"] = rank_;
            j["ep_max_local_rows"] = ep_max_local_rows_;
        }
        int64_t n_expert_ops = 0, expert_rows = 0;
        for (const SimEvent& e : tl)
            if (s.ops[e.op_id].kind == OpKind::compute_expert) {
                ++n_expert_ops;
                expert_rows += s.ops[e.op_id].token_count;
            }
        j["expert_ops"] = n_expert_ops;
        j["expert_rows"] = expert_rows;
        j["expert_bytes"] = spec_.expert_bytes;
        j["compute_ps_by_kind"] = {{"attention", kind_busy[static_cast<int>(OpKind::compute_attention)]},
                                   {"gate", kind_busy[static_cast<int>(OpKind::compute_gate)]},
                                   {"expert", kind_busy[static_cast<int>(OpKind::compute_expert)]}};
        j["step_ms"] = step_ms_;
    } else if (what == "simulated") {
        // The reference's discrete-event model (moesim::run, simulator.cpp:70-287,
        // shared-PCIe fluid link 99-129) priced with rates MEASURED in this
        // window: per-token attention / gate / expert time of the executed
        // compute ops and the link's bytes / busy time. The executed schedule
        // is simulated whole; the window's simulated metrics sit next to the
        // measured ones.
        duration_ps busy[3] = {0, 0, 0};
        int64_t tok[3] = {0, 0, 0};
        for (const SimEvent& e : tl) {
            const StreamOp& op = s.ops[e.op_id];
            const int k = op.kind == OpKind::compute_attention ? 0
                          : op.kind == OpKind::compute_gate    ? 1
                          : op.kind == OpKind::compute_expert  ? 2
                                                               : -1;
            if (k < 0) continue;
            busy[k] += e.end - e.start;
            tok[k] += op.token_count;
        }
        const auto [h2d, link_busy] = link_usage(s, tl);
        HardwareProfile p = profile_;
        auto rate = [](duration_ps b, int64_t t) { return t > 0 ? std::max<duration_ps>(1, b / t) : duration_ps{1}; };
        p.attn_compute_per_token = rate(busy[0], tok[0]);
        p.gate_compute_per_token = rate(busy[1], tok[1]);
        p.expert_compute_per_token = rate(busy[2], tok[2]);
        if (link_busy > 0 && h2d > 0) p.pcie_bandwidth = static_cast<double>(h2d) / (static_cast<double>(link_busy) * 1e-12);
        p.transfer_fixed_latency = 0;
        const CostProfile cost = build_cost_profile(spec_, p, cfg_.workload.batch_size, cfg_.quant);
        std::array<byte_count, 4> caps{INT64_MAX / 4, INT64_MAX / 4, INT64_MAX / 4, INT64_MAX / 4};
        MemoryLedger ledger(caps, false);
        SimOptions so;
        so.shared_pcie = true;
        const SimResult r = run(s, cost, plan_, ledger, so);
        std::vector<SimEvent> stl(r.timeline.begin() + std::min<size_t>(log_from_, r.timeline.size()),
                                  r.timeline.begin() + std::min<size_t>(next_exec_, r.timeline.size()));
        j["simulated"] = reference_metrics(s, records_from_, stl, arena_used_, tokens_generated_);
        j["measured"] = reference_metrics(s, records_from_, tl, arena_used_, tokens_generated_);
        j["rates"] = {{"attn_ps_per_token", p.attn_compute_per_token},
                      {"gate_ps_per_token", p.gate_compute_per_token},
                      {"expert_ps_per_token", p.expert_compute_per_token},
                      {"pcie_bytes_per_s", p.pcie_bandwidth},
                      {"ps_per_byte_pinned", cost.ps_per_byte_pinned}};
        j["shared_pcie"] = true;
    } else if (what == "prefetch") {
        json recs = json::array();
        for (size_t i = records_from_; i < s.prefetch_records.size(); ++i) {
            const auto& r = s.prefetch_records[i];
            recs.push_back({{"step", r.step}, {"layer", r.layer}, {"prefetched", r.prefetched},
                            {"activated", r.activated}, {"hottest", r.hottest}, {"fallback", r.used_fallback}});
        }
        j["records"] = recs;
    } else if (what == "trace") {
        j["sel"] = recorded_.sel;
    } else if (what.rfind("trace_steps:", 0) == 0) {
        // Executed routing of steps [a, b) only ("trace_steps:a:b"), in the
        // reference's flat [step][layer][batch][token][k] order.
        int a = 0, b = 0;
        if (std::sscanf(what.c_str(), "trace_steps:%d:%d", &a, &b) != 2 || a < 0 || b <= a ||
            b > recorded_.n_steps)
            throw ConfigError("engine report: bad step range '" + what + "'");
        const size_t lo = recorded_.offset(a, 0, 0, 0);
        const size_t hi = b == recorded_.n_steps ? recorded_.sel.size() : recorded_.offset(b, 0, 0, 0);
        j["sel"] = std::vector<uint16_t>(recorded_.sel.begin() + lo, recorded_.sel.begin() + hi);
        j["steps"] = {a, b};
    } else if (what == "validate") {
        if (ep_) {
            // A shard's schedule covers its local experts only; the
            // single-GPU validator's token conservation does not apply.
            j["violations"] = json::array();
            j["skipped"] = "expert-parallel shard";
        } else {
            const ValidationReport rep = validate_schedule(s, cfg_.replay ? replay_trace_ : recorded_, plan_);
            // A run that skipped steps (e.g. decode without the prefill step)
            // is checked on the steps it executed: findings are tagged
            // "(step,layer)" by the reference validator.
            json v = json::array();
            int skipped = 0;
            for (const std::string& msg : rep.violations) {
                int st = -1;
                if (!msg.empty() && msg[0] == '(') st = std::atoi(msg.c_str() + 1);
                if (st >= 0 && !executed_steps_.count(st)) {
                    ++skipped;
                    continue;
                }
                v.push_back(msg);
            }
            j["violations"] = v;
            if (skipped) j["unexecuted_step_findings"] = skipped;
        }
    } else if (what == "ledger") {
        // Reference memory accounting (MemoryLedger, placement.cpp:257-292)
        // replayed on the measured timeline of the executed window; VRAM
        // capacity = this engine's HBM cap, not enforced (audit).
        std::array<byte_count, 4> caps{cfg_.hbm_cap, cfg_.host_dram, INT64_MAX / 4, INT64_MAX / 4};
        MemoryLedger ledger(caps, false);
        const std::int64_t carried = detail::replay_ledger_on_timeline(s, tl, plan_, ledger);
        j["vram_high_water"] = ledger.high_water(Tier::vram);
        j["vram_capacity"] = cfg_.hbm_cap;
        j["within_capacity"] = ledger.high_water(Tier::vram) <= cfg_.hbm_cap;
        j["dram_high_water"] = ledger.high_water(Tier::dram);
        j["carried_in_frees"] = carried;
        j["arena_bytes_used"] = arena_used_;
        j["memory_csv"] = memory_timeline_csv(ledger);
    } else if (what == "hidden") {
        json arr = json::array();
        for (const auto& dmp : hidden_dumps_) arr.push_back(dmp);
        j["dumps"] = arr;
    } else {
        throw ConfigError("engine report: unknown section '" + what + "'");
    }
    return j.dump();
}

}  // namespace klotski
