// SPDX-License-Identifier: Apache-2.0
// Incremental Algorithm-1 emitter (internal header).
//
// The reference builds a whole Schedule ahead of time from a pre-drawn trace
// (proj/src/schedule.cpp:466-634). Here the per-block logic is split at the
// one point where it needs routing information:
//   open_block()  : weight bundle (gate + predicted hot experts), next-layer
//                   attention load, n attentions (+KV traffic), n gates;
//   close_block() : cold loads in first-demand order, expert computes
//                   (hot by load, then colds in one reorder group), offloads,
//                   prefetch record, window advance.
// The offline builders call both back to back with routing taken from the
// trace; the B200 engine calls open_block(), launches those ops, reads the
// gate outputs back and then calls close_block() with the device routing —
// so both produce the identical op log for identical routing.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "moesim/schedule.hpp"

namespace moesim::detail {

// Routing facts one block needs, derived from a trace or read back from HBM.
struct BlockRouting {
    std::vector<std::int64_t> group_hist;           // [E] routed rows over the group
    std::vector<std::vector<int>> demand;           // per batch: ids in first-appearance order
    std::vector<std::vector<std::int64_t>> batch_hist;  // per batch: [E]
};

BlockRouting routing_from_trace(const ActivationTrace& trace, int step, int layer);

// Geometry of the batch group being scheduled.
struct GroupShape {
    int n_steps = 0, n_layers = 0, n_batches = 0, batch_size = 0, prompt_len = 0;
    int top_k = 0, n_experts = 0;
    int tokens_per_batch(int step) const { return batch_size * (step == 0 ? prompt_len : 1); }
    static GroupShape of(const ActivationTrace& t) {
        return {t.n_steps, t.n_layers, t.n_batches, t.batch_size, t.prompt_len, t.top_k, t.n_experts};
    }
};

// Op ids of one open block that close_block() needs.
struct OpenBlock {
    int step = 0, layer = 0;
    std::int32_t issue_dep = -1;
    std::vector<int> hot_ids;
    bool fallback = false;
    std::int32_t moe_load = -1, gate_load = -1, next_attn_load = -1;
    std::map<int, std::int32_t> expert_load_op;
    std::vector<std::int32_t> attn, gates;
    // Op ids in emission order, grouped for the executor.
    std::int32_t first_op = 0;
};

// One row of the simple (row-by-row) variant, split at its gate like a block.
struct SimpleRow {
    int step = 0, batch = 0, layer = 0;
    std::int32_t issue = -1, moe = -1, gate = -1, next_attn = -1;
};

struct ClosedBlock {
    std::vector<std::pair<int, int>> cold;  // (expert, demanding batch) in issue order
    std::int32_t block_last = -1;
    std::int32_t first_op = 0;
};

class Emitter {
  public:
    Emitter(Variant v, const PipelinePlan& plan, const GroupShape& shape, const ScheduleOptions& opts);

    // Grouped variants (multibatch_full_prefetch, strawman, klotski).
    OpenBlock open_block(int step, int layer, const PrefetchDecision* decision);
    ClosedBlock close_block(OpenBlock& blk, const BlockRouting& routing);

    // simple variant: one (step, batch, layer) row; open = weights, cache,
    // attention and gate; close = the batch's expert computes (needs routing).
    SimpleRow simple_open(int step, int batch, int layer);
    void simple_close(const SimpleRow& row, const BlockRouting& routing);
    void simple_row(int step, int batch, int layer, const BlockRouting& routing);

    const Schedule& schedule() const { return s_; }
    Schedule take() { return std::move(s_); }
    bool split_moe() const { return split_moe_; }

  private:
    std::int32_t push(StreamOp op);
    bool experts_resident(int layer) const;
    bool attention_resident(int layer) const;
    bool gate_resident(int layer) const;
    bool kv_offloaded() const;
    std::int32_t staged_by(TensorClass cls, int layer) const;

    std::int32_t load_attention(int step, int layer, std::int32_t after);
    std::int32_t load_gate(int step, int layer, std::int32_t after);
    std::int32_t load_moe(int step, int layer, int batch, std::int32_t after);
    void offload_weights(TensorClass cls, int step, int layer, int batch, std::int32_t after);
    std::int32_t load_expert(StreamId stream, int step, int layer, int expert, bool hot,
                             std::vector<std::int32_t> deps);
    void offload_expert(int step, int layer, int expert, std::int32_t after);
    std::int32_t load_kv(int step, int layer, int batch, std::int32_t backpressure);
    void store_kv(int step, int layer, int batch, std::int32_t attn);
    std::int32_t attention(int step, int layer, int batch, std::int32_t weights, std::int32_t cache);
    std::int32_t gate(int step, int layer, int batch, std::int32_t weights, std::int32_t attn);
    std::int32_t expert(int step, int layer, int e, std::int64_t tokens, bool hot, int batch,
                        std::int32_t load, std::int32_t gate_dep, std::int32_t group);
    void advance_window(int step, int layer, std::int32_t after);
    void stage_prologue();

    std::size_t kv_slot(int layer, int batch) const {
        return static_cast<std::size_t>(layer) * shape_.n_batches + batch;
    }

    Variant variant_;
    bool split_moe_;
    const PipelinePlan& plan_;
    GroupShape shape_;
    ScheduleOptions opts_;
    Schedule s_;
    std::vector<std::int32_t> staged_;                   // latest window_stage per layer
    std::vector<std::vector<std::int32_t>> pass_loads_;  // loads of the current pass per layer
    std::vector<std::int32_t> kv_last_store_;
    std::vector<char> kv_host_live_;
    std::int32_t next_group_ = 0;
    // cross-block chaining state
    std::int32_t prev_block_last_ = -1;
    std::int32_t prev_gate_last_ = -1;
    std::int32_t pending_attn_load_ = -1;
};

}  // namespace moesim::detail
