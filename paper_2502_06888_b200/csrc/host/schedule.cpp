// SPDX-License-Identifier: Apache-2.0
// Algorithm 1 (expert-aware multi-batch schedule), its baselines, the table
// prefetcher plugin and the structural validator.
// Semantics: reference proj/src/schedule.cpp (prefetcher 60-91, emission
// helpers 155-426, build_grouped 466-634, build_simple 638-690, to_text
// 706-727, validate_schedule 729-860). Structure differs: see emitter.hpp.
#include <algorithm>
#include <memory>
#include <set>
#include <sstream>

#include "emitter.hpp"
#include "moesim/schedule.hpp"

namespace moesim {

const char* variant_name(Variant v) {
    switch (v) {
        case Variant::simple: return "simple";
        case Variant::multibatch_full_prefetch: return "multibatch_full_prefetch";
        case Variant::strawman_no_reorder: return "strawman_no_reorder";
        case Variant::klotski: return "klotski";
    }
    return "?";
}

Variant variant_from_name(const std::string& name) {
    for (Variant v : {Variant::simple, Variant::multibatch_full_prefetch,
                      Variant::strawman_no_reorder, Variant::klotski})
        if (name == variant_name(v)) return v;
    throw ConfigError("unknown schedule variant '" + name + "'");
}

const char* stream_name(StreamId s) {
    static const char* const names[] = {"compute",     "weight_load", "expert_load",
                                        "cache_load",  "cache_store", "cpu_stage"};
    const int i = static_cast<int>(s);
    return i >= 0 && i < kNumStreams ? names[i] : "?";
}

const char* op_kind_name(OpKind k) {
    static const char* const names[] = {
        "compute_attention", "compute_gate",   "compute_expert", "load_weights",
        "load_expert",       "load_cache",     "store_cache",    "load_hidden",
        "store_hidden",      "offload_expert", "offload_weights", "window_stage"};
    const int i = static_cast<int>(k);
    return i >= 0 && i < 12 ? names[i] : "?";
}

// Table-backed prefetcher with the reference's online-update timing: the call
// for (step, j>0) first folds the transition that produced layer j-1's
// selections into the table (marginal when j-1 == 0), then predicts layer j.
// The transition into the last layer is therefore never folded.
PrefetchProvider make_table_prefetcher(CorrelationTable table, bool online_update,
                                       TendencyAggregation agg, int top_k) {
    struct Memory {
        CorrelationTable table;
        std::vector<std::uint16_t> last_prev;  // selections one layer back
        int last_layer = -1;
        int step = -1;
    };
    auto mem = std::make_shared<Memory>();
    mem->table = std::move(table);
    return [mem, online_update, agg, top_k](int step, int layer,
                                            std::span<const std::uint16_t> prev) {
        if (step != mem->step) {
            mem->step = step;
            mem->last_prev.clear();
            mem->last_layer = -1;
        }
        if (online_update && layer > 0 && !prev.empty()) {
            if (layer == 1)
                update_table(mem->table, 0, {}, prev, top_k);
            else if (mem->last_layer == layer - 1)
                update_table(mem->table, layer - 1, mem->last_prev, prev, top_k);
            mem->last_prev.assign(prev.begin(), prev.end());
            mem->last_layer = layer;
        }
        return predict_hot(mem->table, layer, prev, std::min(top_k, mem->table.n_experts), agg, top_k);
    };
}

namespace detail {

namespace {

std::string weight_tag(TensorClass cls, int step, int layer, int batch = -1) {
    const char c = cls == TensorClass::attention ? 'a' : cls == TensorClass::gate ? 'g' : 'm';
    std::string t = "w:";
    t += c;
    t += ":" + std::to_string(step) + ":" + std::to_string(layer);
    if (batch >= 0) t += ":" + std::to_string(batch);
    return t;
}

std::string expert_tag(int step, int layer, int e) {
    return "e:" + std::to_string(step) + ":" + std::to_string(layer) + ":" + std::to_string(e);
}

std::string kv_tag(const char* kind, int step, int layer, int batch) {
    return std::string(kind) + ":" + std::to_string(step) + ":" + std::to_string(layer) + ":" +
           std::to_string(batch);
}

LedgerEffect alloc_effect(LedgerEffect::When w, Tier t, byte_count b, std::string tag) {
    return {w, true, t, b, std::move(tag)};
}
LedgerEffect free_effect(LedgerEffect::When w, Tier t, std::string tag) {
    return {w, false, t, 0, std::move(tag)};
}

StreamOp make_op(StreamId st, OpKind k, Phase ph, int step, int layer, int batch = -1,
                 int expert = -1) {
    StreamOp op;
    op.stream = st;
    op.kind = k;
    op.phase = ph;
    op.step = static_cast<std::int16_t>(step);
    op.layer = static_cast<std::int16_t>(layer);
    op.batch = static_cast<std::int16_t>(batch);
    op.expert = static_cast<std::int16_t>(expert);
    return op;
}

}  // namespace

BlockRouting routing_from_trace(const ActivationTrace& trace, int step, int layer) {
    BlockRouting r;
    const int E = trace.n_experts;
    r.group_hist = expert_load(trace, step, layer).tokens_per_expert;
    r.demand.resize(trace.n_batches);
    r.batch_hist.assign(trace.n_batches, std::vector<std::int64_t>(E, 0));
    for (int b = 0; b < trace.n_batches; ++b)
        for (std::uint16_t e : trace.batch_selections(step, layer, b))
            if (r.batch_hist[b][e]++ == 0) r.demand[b].push_back(e);
    return r;
}

Emitter::Emitter(Variant v, const PipelinePlan& plan, const GroupShape& shape,
                 const ScheduleOptions& opts)
    : variant_(v),
      split_moe_(v == Variant::klotski || v == Variant::strawman_no_reorder),
      plan_(plan),
      shape_(shape),
      opts_(opts) {
    s_.variant = v;
    s_.n_steps = shape.n_steps;
    s_.n_layers = shape.n_layers;
    s_.n_batches = shape.n_batches;
    s_.batch_size = shape.batch_size;
    s_.top_k = shape.top_k;
    s_.n_experts = shape.n_experts;
    staged_.assign(shape.n_layers, -1);
    pass_loads_.resize(shape.n_layers);
    kv_last_store_.assign(static_cast<std::size_t>(shape.n_layers) * shape.n_batches, -1);
    kv_host_live_.assign(kv_last_store_.size(), 0);
    stage_prologue();
    if (!attention_resident(0)) pending_attn_load_ = load_attention(0, 0, -1);
}

std::int32_t Emitter::push(StreamOp op) {
    op.id = static_cast<std::int32_t>(s_.ops.size());
    auto& d = op.deps;
    d.erase(std::remove_if(d.begin(), d.end(), [](std::int32_t x) { return x < 0; }), d.end());
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    s_.streams[static_cast<int>(op.stream)].push_back(op.id);
    s_.ops.push_back(std::move(op));
    return s_.ops.back().id;
}

bool Emitter::experts_resident(int l) const { return plan_.placement.expert_tier[l] == Tier::vram; }
bool Emitter::attention_resident(int l) const { return plan_.placement.attention_tier[l] == Tier::vram; }
bool Emitter::gate_resident(int l) const { return plan_.placement.gate_tier[l] == Tier::vram; }
bool Emitter::kv_offloaded() const { return plan_.placement.kv_tier != Tier::vram; }

std::int32_t Emitter::staged_by(TensorClass cls, int l) const {
    const auto& pl = plan_.placement;
    const Tier t = cls == TensorClass::expert ? pl.expert_tier[l]
                   : cls == TensorClass::gate ? pl.gate_tier[l]
                                              : pl.attention_tier[l];
    return t == Tier::disk ? staged_[l] : -1;
}

std::int32_t Emitter::load_attention(int step, int layer, std::int32_t after) {
    StreamOp op = make_op(StreamId::weight_load, OpKind::load_weights, Phase::other, step, layer);
    op.cls = TensorClass::attention;
    op.payload_bytes = plan_.cost.attention_transfer_bytes;
    op.deps = {after, staged_by(TensorClass::attention, layer)};
    op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::vram,
                                     plan_.model.attention_bytes,
                                     weight_tag(TensorClass::attention, step, layer)));
    const std::int32_t id = push(std::move(op));
    pass_loads_[layer].push_back(id);
    return id;
}

std::int32_t Emitter::load_gate(int step, int layer, std::int32_t after) {
    StreamOp op = make_op(StreamId::weight_load, OpKind::load_weights, Phase::other, step, layer);
    op.cls = TensorClass::gate;
    op.payload_bytes = plan_.cost.gate_transfer_bytes;
    op.deps = {after, staged_by(TensorClass::gate, layer)};
    op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::vram, plan_.model.gate_bytes,
                                     weight_tag(TensorClass::gate, step, layer)));
    const std::int32_t id = push(std::move(op));
    pass_loads_[layer].push_back(id);
    return id;
}

std::int32_t Emitter::load_moe(int step, int layer, int batch, std::int32_t after) {
    StreamOp op = make_op(StreamId::weight_load, OpKind::load_weights, Phase::other, step, layer, batch);
    op.cls = TensorClass::expert;
    op.payload_bytes = plan_.cost.moe_transfer_bytes;
    op.deps = {after, staged_by(TensorClass::expert, layer), staged_by(TensorClass::gate, layer)};
    op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::vram,
                                     tensor_bytes(plan_.model, TensorKind::moe_layer),
                                     weight_tag(TensorClass::gate, step, layer, batch)));
    const std::int32_t id = push(std::move(op));
    pass_loads_[layer].push_back(id);
    return id;
}

void Emitter::offload_weights(TensorClass cls, int step, int layer, int batch, std::int32_t after) {
    StreamOp op = make_op(StreamId::cache_store, OpKind::offload_weights, Phase::other, step, layer, batch);
    op.cls = cls;
    op.deps = {after};
    op.ledger.push_back(free_effect(LedgerEffect::When::at_start, Tier::vram,
                                    weight_tag(cls, step, layer, batch)));
    push(std::move(op));
}

std::int32_t Emitter::load_expert(StreamId stream, int step, int layer, int e, bool hot,
                                  std::vector<std::int32_t> deps) {
    StreamOp op = make_op(stream, OpKind::load_expert, Phase::expert, step, layer, -1, e);
    op.cls = TensorClass::expert;
    op.hot = hot;
    op.payload_bytes = plan_.cost.expert_transfer_bytes;
    op.deps = std::move(deps);
    op.deps.push_back(staged_by(TensorClass::expert, layer));
    op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::vram, plan_.model.expert_bytes,
                                     expert_tag(step, layer, e)));
    const std::int32_t id = push(std::move(op));
    pass_loads_[layer].push_back(id);
    return id;
}

void Emitter::offload_expert(int step, int layer, int e, std::int32_t after) {
    StreamOp op = make_op(StreamId::cache_store, OpKind::offload_expert, Phase::expert, step, layer, -1, e);
    op.cls = TensorClass::expert;
    op.deps = {after};
    op.ledger.push_back(free_effect(LedgerEffect::When::at_start, Tier::vram, expert_tag(step, layer, e)));
    push(std::move(op));
}

std::int32_t Emitter::load_kv(int step, int layer, int batch, std::int32_t backpressure) {
    if (!kv_offloaded() || step == 0) return -1;
    const int history = plan_.placement.kv_retention.retained(shape_.prompt_len + step - 1);
    StreamOp op = make_op(StreamId::cache_load, OpKind::load_cache, Phase::attention, step, layer, batch);
    op.cls = TensorClass::kv_cache;
    op.payload_bytes =
        static_cast<byte_count>(history) * shape_.batch_size * plan_.model.kv_bytes_per_token;
    op.route = plan_.placement.kv_tier == Tier::disk ? TransferRoute::disk_dram
                                                     : TransferRoute::dram_vram_unpinned;
    op.deps = {kv_last_store_[kv_slot(layer, batch)], backpressure};
    op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::vram, op.payload_bytes,
                                     kv_tag("kvl", step, layer, batch)));
    return push(std::move(op));
}

void Emitter::store_kv(int step, int layer, int batch, std::int32_t attn) {
    if (!kv_offloaded()) return;
    StreamOp op = make_op(StreamId::cache_store, OpKind::store_cache, Phase::attention, step, layer, batch);
    op.cls = TensorClass::kv_cache;
    op.payload_bytes =
        static_cast<byte_count>(shape_.tokens_per_batch(step)) * plan_.model.kv_bytes_per_token;
    op.route = TransferRoute::vram_dram;
    op.deps = {attn};
    op.ledger.push_back(free_effect(LedgerEffect::When::at_end, Tier::vram, kv_tag("kvn", step, layer, batch)));
    const std::size_t slot = kv_slot(layer, batch);
    const std::string host_tag = "kvd:" + std::to_string(layer) + ":" + std::to_string(batch);
    if (kv_host_live_[slot]) op.ledger.push_back(free_effect(LedgerEffect::When::at_end, Tier::dram, host_tag));
    const int kept = plan_.placement.kv_retention.retained(shape_.prompt_len + step);
    op.ledger.push_back(alloc_effect(
        LedgerEffect::When::at_end, Tier::dram,
        static_cast<byte_count>(kept) * shape_.batch_size * plan_.model.kv_bytes_per_token, host_tag));
    kv_host_live_[slot] = 1;
    kv_last_store_[slot] = push(std::move(op));
}

std::int32_t Emitter::attention(int step, int layer, int batch, std::int32_t weights,
                                std::int32_t cache) {
    StreamOp op = make_op(StreamId::compute, OpKind::compute_attention, Phase::attention, step, layer, batch);
    op.cls = TensorClass::attention;
    op.token_count = shape_.tokens_per_batch(step);
    op.deps = {weights, cache};
    const byte_count fresh = static_cast<byte_count>(shape_.tokens_per_batch(step)) * plan_.model.kv_bytes_per_token;
    if (kv_offloaded()) {
        op.ledger.push_back(alloc_effect(LedgerEffect::When::at_end, Tier::vram, fresh,
                                         kv_tag("kvn", step, layer, batch)));
        if (cache >= 0)
            op.ledger.push_back(free_effect(LedgerEffect::When::at_end, Tier::vram, kv_tag("kvl", step, layer, batch)));
    } else {
        op.ledger.push_back(alloc_effect(LedgerEffect::When::at_end, Tier::vram, fresh,
                                         kv_tag("kvr", step, layer, batch)));
    }
    return push(std::move(op));
}

std::int32_t Emitter::gate(int step, int layer, int batch, std::int32_t weights, std::int32_t attn) {
    StreamOp op = make_op(StreamId::compute, OpKind::compute_gate, Phase::gate, step, layer, batch);
    op.cls = TensorClass::gate;
    op.token_count = shape_.tokens_per_batch(step);
    op.deps = {weights, attn};
    return push(std::move(op));
}

std::int32_t Emitter::expert(int step, int layer, int e, std::int64_t tokens, bool hot, int batch,
                             std::int32_t load, std::int32_t gate_dep, std::int32_t group) {
    StreamOp op = make_op(StreamId::compute, OpKind::compute_expert, Phase::expert, step, layer, batch, e);
    op.cls = TensorClass::expert;
    op.token_count = tokens;
    op.hot = hot;
    op.reorder_group = group;
    op.deps = {load, gate_dep};
    return push(std::move(op));
}

void Emitter::advance_window(int step, int layer, std::int32_t after) {
    const auto& pl = plan_.placement;
    if (pl.cpu_window_L > 0) {
        for (const StageIntent& in : window_advance(pl, layer)) {
            const byte_count in_bytes = pl.disk_bytes_of_layer(in.stage_layer, plan_.model, plan_.quant);
            const byte_count out_bytes = pl.disk_bytes_of_layer(in.evict_layer, plan_.model, plan_.quant);
            if (in_bytes == 0 && out_bytes == 0) continue;
            StreamOp op = make_op(StreamId::cpu_stage, OpKind::window_stage, Phase::other, step,
                                  in.stage_layer, in.evict_layer);
            op.payload_bytes = in_bytes;
            op.route = TransferRoute::disk_dram;
            op.deps = {after};
            op.deps.insert(op.deps.end(), pass_loads_[in.evict_layer].begin(),
                           pass_loads_[in.evict_layer].end());
            if (out_bytes > 0)
                op.ledger.push_back(free_effect(LedgerEffect::When::at_start, Tier::dram,
                                                "stg:" + std::to_string(in.evict_layer)));
            if (in_bytes > 0)
                op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::dram, in_bytes,
                                                 "stg:" + std::to_string(in.stage_layer)));
            const std::int32_t id = push(std::move(op));
            if (in_bytes > 0) staged_[in.stage_layer] = id;
        }
    }
    pass_loads_[layer].clear();
}

void Emitter::stage_prologue() {
    const auto& pl = plan_.placement;
    for (int l = 0; l < pl.cpu_window_L && l < shape_.n_layers; ++l) {
        const byte_count bytes = pl.disk_bytes_of_layer(l, plan_.model, plan_.quant);
        if (bytes == 0) continue;
        StreamOp op = make_op(StreamId::cpu_stage, OpKind::window_stage, Phase::other, 0, l);
        op.payload_bytes = bytes;
        op.route = TransferRoute::disk_dram;
        op.ledger.push_back(alloc_effect(LedgerEffect::When::at_start, Tier::dram, bytes,
                                         "stg:" + std::to_string(l)));
        staged_[l] = push(std::move(op));
    }
}

OpenBlock Emitter::open_block(int step, int layer, const PrefetchDecision* decision) {
    OpenBlock b;
    b.step = step;
    b.layer = layer;
    b.issue_dep = prev_block_last_;
    b.first_op = static_cast<std::int32_t>(s_.ops.size());
    const int n = shape_.n_batches;

    // Weight-stream bundle: gate + predicted hot experts (Eq. 2 overlap with
    // this block's attentions), or the whole MoE layer for the baselines.
    if (split_moe_) {
        if (decision == nullptr) throw ConfigError("hot-prefetch variants need a prefetch provider");
        for (int e : decision->expert_ids)
            if (e < 0 || e >= shape_.n_experts)
                throw ValidationError("prefetch provider returned expert id " + std::to_string(e) +
                                      " out of range");
        b.hot_ids = decision->expert_ids;
        b.fallback = decision->used_fallback;
        if (!gate_resident(layer)) b.gate_load = load_gate(step, layer, b.issue_dep);
        if (!experts_resident(layer))
            for (int e : b.hot_ids)
                b.expert_load_op[e] = load_expert(StreamId::weight_load, step, layer, e, true,
                                                  {b.issue_dep, layer > 0 ? prev_gate_last_ : -1});
    } else if (!experts_resident(layer) || !gate_resident(layer)) {
        b.moe_load = load_moe(step, layer, -1, b.issue_dep);
        b.gate_load = b.moe_load;
    }

    // Next block's attention weights (Alg. 1 lines 3-4).
    const bool last_layer = layer + 1 >= shape_.n_layers;
    const int nl = last_layer ? 0 : layer + 1;
    const int ns = last_layer ? step + 1 : step;
    if (ns < shape_.n_steps && !attention_resident(nl)) b.next_attn_load = load_attention(ns, nl, b.issue_dep);

    // n attentions with double-buffered KV loads.
    b.attn.assign(n, -1);
    for (int k = 0; k < n; ++k) {
        const std::int32_t cache = load_kv(step, layer, k, k >= 2 ? b.attn[k - 2] : -1);
        b.attn[k] = attention(step, layer, k, pending_attn_load_, cache);
        store_kv(step, layer, k, b.attn[k]);
    }
    if (pending_attn_load_ >= 0) offload_weights(TensorClass::attention, step, layer, -1, b.attn[n - 1]);

    b.gates.assign(n, -1);
    for (int k = 0; k < n; ++k) b.gates[k] = gate(step, layer, k, b.gate_load, b.attn[k]);
    return b;
}

ClosedBlock Emitter::close_block(OpenBlock& b, const BlockRouting& r) {
    ClosedBlock c;
    c.first_op = static_cast<std::int32_t>(s_.ops.size());
    const int n = shape_.n_batches, step = b.step, layer = b.layer;
    const std::int32_t last_gate = b.gates[n - 1];
    const auto& hist = r.group_hist;

    // Cold experts: first demand across batches 0..n-1, minus the hot set;
    // each transfer waits for the gate of the batch that first demanded it.
    if (split_moe_) {
        std::set<int> seen(b.hot_ids.begin(), b.hot_ids.end());
        for (int k = 0; k < n; ++k)
            for (int e : r.demand[k])
                if (seen.insert(e).second) c.cold.emplace_back(e, k);
        if (!experts_resident(layer))
            for (const auto& [e, k] : c.cold)
                b.expert_load_op[e] = load_expert(StreamId::expert_load, step, layer, e, false, {b.gates[k]});
    }

    std::vector<std::int32_t> last_use(shape_.n_experts, -1);
    std::int32_t block_last = last_gate;
    auto load_of = [&](int e) -> std::int32_t {
        if (b.moe_load >= 0) return b.moe_load;
        const auto it = b.expert_load_op.find(e);
        return it == b.expert_load_op.end() ? -1 : it->second;
    };

    if (variant_ == Variant::klotski) {
        // Expert-major: active hot experts by routed rows (desc, id asc), then
        // the colds in transfer order sharing one reorder group.
        std::vector<int> hot;
        for (int e : b.hot_ids)
            if (hist[e] > 0) hot.push_back(e);
        std::stable_sort(hot.begin(), hot.end(), [&](int x, int y) {
            return hist[x] != hist[y] ? hist[x] > hist[y] : x < y;
        });
        for (int e : hot) last_use[e] = block_last = expert(step, layer, e, hist[e], true, -1, load_of(e), last_gate, -1);
        const std::int32_t group = c.cold.size() > 1 ? next_group_++ : -1;
        for (const auto& [e, k] : c.cold)
            last_use[e] = block_last = expert(step, layer, e, hist[e], false, -1, load_of(e), last_gate, group);
    } else {
        // Batch-major computes (the stall the reorder removes).
        const std::set<int> hotset(b.hot_ids.begin(), b.hot_ids.end());
        for (int k = 0; k < n; ++k)
            for (int e : r.demand[k]) {
                const bool hot = split_moe_ && hotset.count(e) > 0;
                last_use[e] = block_last =
                    expert(step, layer, e, r.batch_hist[k][e], hot, k, load_of(e), b.gates[k], -1);
            }
    }

    if (split_moe_ && !experts_resident(layer))
        for (const auto& [e, id] : b.expert_load_op) {
            std::int32_t after = last_use[e];
            if (!opts_.immediate_offload || after < 0) after = block_last;
            offload_expert(step, layer, e, after);
        }
    if (b.moe_load >= 0) offload_weights(TensorClass::gate, step, layer, -1, block_last);
    if (split_moe_ && b.gate_load >= 0) offload_weights(TensorClass::gate, step, layer, -1, last_gate);

    if (split_moe_) {
        LayerPrefetchRecord rec;
        rec.step = step;
        rec.layer = layer;
        rec.prefetched = b.hot_ids;
        for (int e = 0; e < shape_.n_experts; ++e)
            if (hist[e] > 0) rec.activated.push_back(e);
        ExpertLoad load;
        load.tokens_per_expert = hist;
        rec.hottest = load.by_hotness();
        if (static_cast<int>(rec.hottest.size()) > plan_.K) rec.hottest.resize(plan_.K);
        rec.used_fallback = b.fallback;
        s_.prefetch_records.push_back(std::move(rec));
    }
    s_.sync_points.emplace_back(step, layer);
    advance_window(step, layer, b.issue_dep);
    prev_block_last_ = block_last;
    prev_gate_last_ = last_gate;
    pending_attn_load_ = b.next_attn_load;
    c.block_last = block_last;
    return c;
}

SimpleRow Emitter::simple_open(int step, int batch, int layer) {
    SimpleRow row{step, batch, layer, prev_block_last_, -1, -1, -1};
    if (!experts_resident(layer) || !gate_resident(layer)) row.moe = load_moe(step, layer, batch, row.issue);

    // Next row in (step, batch, layer) order.
    int nl = layer + 1, nb = batch, ns = step;
    if (nl == shape_.n_layers) {
        nl = 0;
        if (++nb == shape_.n_batches) {
            nb = 0;
            ++ns;
        }
    }
    if (ns < shape_.n_steps && !attention_resident(nl)) row.next_attn = load_attention(ns, nl, row.issue);

    const std::int32_t cache = load_kv(step, layer, batch, -1);
    const std::int32_t att = attention(step, layer, batch, pending_attn_load_, cache);
    store_kv(step, layer, batch, att);
    if (pending_attn_load_ >= 0) offload_weights(TensorClass::attention, step, layer, -1, att);
    row.gate = gate(step, layer, batch, row.moe, att);
    return row;
}

void Emitter::simple_close(const SimpleRow& row, const BlockRouting& r) {
    std::int32_t last = row.gate;
    for (int e : r.demand[row.batch])
        last = expert(row.step, row.layer, e, r.batch_hist[row.batch][e], false, row.batch, row.moe, row.gate, -1);
    if (row.moe >= 0) offload_weights(TensorClass::gate, row.step, row.layer, row.batch, last);
    s_.sync_points.emplace_back(row.step, row.layer);
    advance_window(row.step, row.layer, row.issue);
    prev_block_last_ = last;
    pending_attn_load_ = row.next_attn;
}

void Emitter::simple_row(int step, int batch, int layer, const BlockRouting& r) {
    simple_close(simple_open(step, batch, layer), r);
}

}  // namespace detail

namespace {

Schedule build_grouped_offline(Variant v, const PipelinePlan& plan, const ActivationTrace& trace,
                               const PrefetchProvider& prefetch, const ScheduleOptions& opts) {
    const bool split = v == Variant::klotski || v == Variant::strawman_no_reorder;
    if (split && !prefetch) throw ConfigError("hot-prefetch variants need a prefetch provider");
    detail::Emitter em(v, plan, detail::GroupShape::of(trace), opts);
    for (int step = 0; step < trace.n_steps; ++step)
        for (int layer = 0; layer < trace.n_layers; ++layer) {
            const detail::BlockRouting routing = detail::routing_from_trace(trace, step, layer);
            PrefetchDecision d;
            if (split) {
                std::span<const std::uint16_t> prev;
                if (layer > 0) prev = trace.layer_selections(step, layer - 1);
                d = prefetch(step, layer, prev);
            }
            detail::OpenBlock blk = em.open_block(step, layer, split ? &d : nullptr);
            em.close_block(blk, routing);
        }
    return em.take();
}

}  // namespace

Schedule build_klotski_schedule(const PipelinePlan& plan, const ActivationTrace& trace,
                                const PrefetchProvider& prefetch, const ScheduleOptions& opts) {
    return build_grouped_offline(Variant::klotski, plan, trace, prefetch, opts);
}

Schedule build_baseline_schedule(Variant variant, const PipelinePlan& plan,
                                 const ActivationTrace& trace, const PrefetchProvider& prefetch,
                                 const ScheduleOptions& opts) {
    if (variant != Variant::simple) return build_grouped_offline(variant, plan, trace, prefetch, opts);
    detail::Emitter em(Variant::simple, plan, detail::GroupShape::of(trace), opts);
    for (int step = 0; step < trace.n_steps; ++step)
        for (int batch = 0; batch < trace.n_batches; ++batch)
            for (int layer = 0; layer < trace.n_layers; ++layer)
                em.simple_row(step, batch, layer, detail::routing_from_trace(trace, step, layer));
    return em.take();
}

std::string Schedule::to_text() const {
    std::ostringstream os;
    os << "schedule variant=" << variant_name(variant) << " steps=" << n_steps << " layers=" << n_layers
       << " batches=" << n_batches << " ops=" << ops.size() << "\n";
    for (const StreamOp& op : ops) {
        os << op.id << " " << stream_name(op.stream) << " " << op_kind_name(op.kind) << " s" << op.step
           << " l" << op.layer;
        if (op.batch >= 0) os << " b" << op.batch;
        if (op.expert >= 0) os << " e" << op.expert;
        if (op.payload_bytes > 0) os << " bytes=" << op.payload_bytes;
        if (op.token_count > 0) os << " tokens=" << op.token_count;
        if (op.hot) os << " hot";
        if (op.reorder_group >= 0) os << " group=" << op.reorder_group;
        os << " deps=[";
        for (std::size_t i = 0; i < op.deps.size(); ++i) os << (i ? "," : "") << op.deps[i];
        os << "]\n";
    }
    return os.str();
}

ValidationReport validate_schedule(const Schedule& s, const ActivationTrace& trace,
                                   const PipelinePlan& plan) {
    ValidationReport rep;
    auto bad = [&](std::string m) { rep.violations.push_back(std::move(m)); };
    const std::int32_t n_ops = static_cast<std::int32_t>(s.ops.size());
    auto in_range = [&](std::int32_t d) { return d >= 0 && d < n_ops; };

    for (std::int32_t i = 0; i < n_ops; ++i) {
        const StreamOp& op = s.ops[i];
        if (op.id != i) bad("op id/index mismatch");
        for (std::int32_t d : op.deps)
            if (!in_range(d)) bad("op " + std::to_string(op.id) + ": dependency out of range");
    }
    std::size_t listed = 0;
    for (int st = 0; st < kNumStreams; ++st) {
        listed += s.streams[st].size();
        for (std::int32_t id : s.streams[st])
            if (s.ops[id].stream != static_cast<StreamId>(st))
                bad("op " + std::to_string(id) + ": listed on the wrong stream");
    }
    if (listed != s.ops.size()) bad("per-stream lists do not cover all ops");

    // Kahn over dependency edges plus per-stream FIFO edges.
    {
        std::vector<int> indeg(n_ops, 0);
        std::vector<std::vector<std::int32_t>> succ(n_ops);
        auto edge = [&](std::int32_t a, std::int32_t b) {
            succ[a].push_back(b);
            ++indeg[b];
        };
        for (const StreamOp& op : s.ops)
            for (std::int32_t d : op.deps)
                if (in_range(d)) edge(d, op.id);
        for (int st = 0; st < kNumStreams; ++st)
            for (std::size_t i = 1; i < s.streams[st].size(); ++i) edge(s.streams[st][i - 1], s.streams[st][i]);
        std::vector<std::int32_t> ready;
        for (std::int32_t i = 0; i < n_ops; ++i)
            if (indeg[i] == 0) ready.push_back(i);
        std::size_t visited = 0;
        while (!ready.empty()) {
            const std::int32_t v = ready.back();
            ready.pop_back();
            ++visited;
            for (std::int32_t w : succ[v])
                if (--indeg[w] == 0) ready.push_back(w);
        }
        if (visited != s.ops.size()) bad("dependency graph has a cycle");
    }

    struct Audit {
        std::map<int, int> loads, offloads;
        std::map<int, std::int64_t> tokens;
    };
    std::map<std::pair<int, int>, Audit> audit;
    for (const StreamOp& op : s.ops) {
        Audit& a = audit[{op.step, op.layer}];
        if (op.kind == OpKind::load_expert) ++a.loads[op.expert];
        else if (op.kind == OpKind::offload_expert) ++a.offloads[op.expert];
        else if (op.kind == OpKind::compute_expert) a.tokens[op.expert] += op.token_count;
    }
    std::map<std::pair<int, int>, std::set<int>> prefetched;
    for (const LayerPrefetchRecord& r : s.prefetch_records)
        prefetched[{r.step, r.layer}].insert(r.prefetched.begin(), r.prefetched.end());
    const bool whole_layer_loads = s.variant == Variant::simple || s.variant == Variant::multibatch_full_prefetch;

    for (int step = 0; step < trace.n_steps; ++step)
        for (int layer = 0; layer < trace.n_layers; ++layer) {
            const ExpertLoad load = expert_load(trace, step, layer);
            Audit& a = audit[{step, layer}];
            const std::set<int>& hot = prefetched[{step, layer}];
            const bool resident = plan.placement.expert_tier[layer] == Tier::vram;
            const std::string where = "(" + std::to_string(step) + "," + std::to_string(layer) + ")";
            const std::int64_t want = static_cast<std::int64_t>(trace.top_k) * trace.tokens_in_step(step);
            std::int64_t got = 0;
            for (const auto& [e, t] : a.tokens) got += t;
            if (got != want)
                bad(where + ": expert compute tokens " + std::to_string(got) + " != top_k * tokens " +
                    std::to_string(want));
            for (int e = 0; e < trace.n_experts; ++e) {
                const bool active = load.tokens_per_expert[e] > 0;
                const int loads = a.loads.count(e) ? a.loads[e] : 0;
                const int offs = a.offloads.count(e) ? a.offloads[e] : 0;
                const bool computed = a.tokens.count(e) > 0;
                const std::string tag = where + " expert " + std::to_string(e);
                if (loads > 1) bad(tag + ": double load");
                if (active && !resident && !whole_layer_loads && loads == 0)
                    bad(tag + ": compute before load (no load op)");
                if (!active && !hot.count(e) && (loads || offs || computed))
                    bad(tag + ": op references an inactive expert");
                if (active && !computed) bad(tag + ": activated expert never computed");
                if (loads != offs) bad(tag + ": loads and offloads unbalanced");
            }
        }

    for (const StreamOp& op : s.ops) {
        if (op.stream != StreamId::compute) continue;
        const auto& pl = plan.placement;
        bool needs = false;
        if (op.kind == OpKind::compute_expert) needs = pl.expert_tier[op.layer] != Tier::vram;
        else if (op.kind == OpKind::compute_gate) needs = pl.gate_tier[op.layer] != Tier::vram;
        else if (op.kind == OpKind::compute_attention) needs = pl.attention_tier[op.layer] != Tier::vram;
        if (!needs) continue;
        const bool has_load = std::any_of(op.deps.begin(), op.deps.end(), [&](std::int32_t d) {
            return in_range(d) && (s.ops[d].kind == OpKind::load_weights || s.ops[d].kind == OpKind::load_expert);
        });
        if (!has_load) bad("op " + std::to_string(op.id) + ": compute before load (missing weight dependency)");
    }
    return rep;
}

}  // namespace moesim
