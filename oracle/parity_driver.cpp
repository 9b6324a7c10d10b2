// Parity driver: one source, compiled twice.
//   * against the reference headers/library with -Dmoesim=moesim_ref
//     -> oracle/_ref/libref_parity.so   (the oracle side)
//   * against this repo's include/moesim + libklotski.so
//     -> paper_2502_06888_b200/libparity.so (the product side)
// Both expose the same extern "C" entry points; tests feed both the same JSON
// request and compare the JSON answers field by field. It exercises the
// reference call stack B (experiment.cpp:183-223): warm-up trace ->
// build_table -> compute_trace_stats -> make_plan -> generate_trace ->
// make_table_prefetcher -> build_*_schedule -> validate_schedule -> run.
//
// Test infrastructure only; never on the product path.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <sstream>
#include <string>

#include <nlohmann/json.hpp>

#include "moesim/correlation.hpp"
#include "moesim/cost.hpp"
#include "moesim/error.hpp"
#include "moesim/model.hpp"
#include "moesim/planner.hpp"
#include "moesim/quant.hpp"
#include "moesim/schedule.hpp"
#include "moesim/simulator.hpp"
#include "moesim/trace.hpp"

using nlohmann::json;

namespace {

moesim::ModelSpec model_of(const json& j) {
    const std::string preset = j.value("preset", "toy");
    moesim::ModelSpec m;
    if (preset == "mixtral-8x7b-like")
        m = moesim::mixtral_8x7b_like();
    else if (preset == "mixtral-8x22b-like")
        m = moesim::mixtral_8x22b_like();
    else
        m = moesim::toy_model(j.value("n_layers", 4), j.value("n_experts", 4), j.value("top_k", 2));
    if (j.contains("n_layers")) m.n_layers = j["n_layers"].get<int>();
    if (j.contains("n_experts")) m.n_experts_per_layer = j["n_experts"].get<int>();
    if (j.contains("top_k")) m.top_k = j["top_k"].get<int>();
    if (j.contains("expert_bytes")) m.expert_bytes = j["expert_bytes"].get<std::int64_t>();
    if (j.contains("attention_bytes")) m.attention_bytes = j["attention_bytes"].get<std::int64_t>();
    if (j.contains("gate_bytes")) m.gate_bytes = j["gate_bytes"].get<std::int64_t>();
    if (j.contains("kv_bytes_per_token"))
        m.kv_bytes_per_token = j["kv_bytes_per_token"].get<std::int64_t>();
    return m;
}

moesim::HardwareProfile hw_of(const json& j) {
    const std::string preset = j.value("preset", "toy-hw");
    moesim::HardwareProfile p = preset == "env1"   ? moesim::env1_profile()
                                : preset == "env2" ? moesim::env2_profile()
                                                   : moesim::toy_profile();
    if (j.contains("vram_capacity")) p.vram_capacity = j["vram_capacity"].get<std::int64_t>();
    if (j.contains("dram_capacity")) p.dram_capacity = j["dram_capacity"].get<std::int64_t>();
    if (j.contains("disk_capacity")) p.disk_capacity = j["disk_capacity"].get<std::int64_t>();
    if (j.contains("pcie_bandwidth")) p.pcie_bandwidth = j["pcie_bandwidth"].get<double>();
    if (j.contains("disk_bandwidth")) p.disk_bandwidth = j["disk_bandwidth"].get<double>();
    if (j.contains("transfer_fixed_latency_ps"))
        p.transfer_fixed_latency = j["transfer_fixed_latency_ps"].get<std::int64_t>();
    if (j.contains("attn_ps")) p.attn_compute_per_token = j["attn_ps"].get<std::int64_t>();
    if (j.contains("gate_ps")) p.gate_compute_per_token = j["gate_ps"].get<std::int64_t>();
    if (j.contains("expert_ps")) p.expert_compute_per_token = j["expert_ps"].get<std::int64_t>();
    if (j.contains("dequant_ps_per_byte"))
        p.dequant_ps_per_byte = j["dequant_ps_per_byte"].get<double>();
    return p;
}

moesim::SkewSpec skew_of(const json& j) {
    const std::string k = j.value("kind", "zipf");
    if (k == "uniform") return moesim::SkewSpec::uniform();
    if (k == "markov") return moesim::SkewSpec::markov(j.value("s", 1.5), j.value("p", 0.8));
    return moesim::SkewSpec::zipf(j.value("s", 1.5));
}

std::uint64_t fnv1a(const std::uint16_t* p, std::size_t n) {
    std::uint64_t h = 1469598103934665603ULL;
    for (std::size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

const char* dup(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

// 4-bit format pins (quant.cpp:120-252): fit_minmax per group and
// dequantize of a flat QuantizedTensor, straight from the library.
json quant_ops(const json& q) {
    json out;
    if (q.contains("fit")) {
        const int bits = q.value("bits", 4);
        json fits = json::array();
        for (const auto& g : q["fit"]) {
            const std::vector<float> v = g.get<std::vector<float>>();
            const moesim::QuantParams p = moesim::fit_minmax(v, bits);
            fits.push_back({p.scale, p.zero});
        }
        out["fit"] = fits;
    }
    if (q.contains("dequant")) {
        const json& d = q["dequant"];
        moesim::QuantizedTensor t;
        t.cfg.bits = d.value("bits", 4);
        t.cfg.group_size = d.value("group_size", 64);
        t.n_elements = d.at("n").get<std::size_t>();
        t.packed = d.at("packed").get<std::vector<std::uint8_t>>();
        t.scales_f16 = d.at("scales").get<std::vector<std::uint16_t>>();
        t.zeros_f16 = d.at("zeros").get<std::vector<std::uint16_t>>();
        out["dequant"] = moesim::dequantize(t);
    }
    if (q.contains("bytes")) {
        moesim::QuantConfig c;
        out["bytes"] = moesim::quantized_bytes(q["bytes"].get<std::int64_t>(), c);
    }
    return out;
}

json request(const char* text) {
    json req = json::parse(text);
    if (req.contains("quant_ops")) return quant_ops(req["quant_ops"]);
    const moesim::ModelSpec model = model_of(req.value("model", json::object()));
    const moesim::HardwareProfile hw = hw_of(req.value("hw", json::object()));
    const json w = req.value("workload", json::object());
    moesim::BatchGroupConfig cfg;
    cfg.batch_size = w.value("batch_size", 4);
    cfg.n_batches = w.value("n_batches", 2);
    cfg.prompt_len = w.value("prompt_len", 4);
    cfg.gen_len = w.value("gen_len", 2);
    const moesim::SkewSpec skew = skew_of(req.value("skew", json::object()));
    const std::uint64_t seed = req.value("seed", 1ULL);
    const std::string variant = req.value("variant", "klotski");
    std::optional<moesim::QuantConfig> quant;
    if (req.value("quant", false)) quant = moesim::QuantConfig{};
    moesim::KvRetentionPolicy retention;
    if (req.value("streaming_kv", false)) retention.mode = moesim::KvRetentionPolicy::Mode::streaming;
    retention.sink_tokens = req.value("sink_tokens", retention.sink_tokens);
    retention.window_tokens = req.value("window_tokens", retention.window_tokens);
    std::optional<int> n_override;
    if (req.contains("n")) n_override = req["n"].get<int>();
    const auto load_model = static_cast<moesim::ExpertLoadModel>(req.value("load_model", 1));
    moesim::PlacementConfig pcfg;
    pcfg.working_set_override = req.value("working_set_override", std::int64_t{0});

    json out;
    // Warm-up trace and table (experiment.cpp prepare: disjoint warm-up seed).
    moesim::BatchGroupConfig warm = cfg;
    warm.n_batches = cfg.batch_size > 1 ? 2 : 4;
    const moesim::ActivationTrace wt = moesim::generate_trace(model, warm, skew, seed + 1);
    const moesim::CorrelationTable table = moesim::build_table(wt, model);
    const moesim::TraceStats stats = moesim::compute_trace_stats(wt, model.top_k);
    out["warm_hash"] = fnv1a(wt.sel.data(), wt.sel.size());
    out["table_text"] = moesim::table_to_string(table);

    const moesim::PipelinePlan plan =
        moesim::make_plan(model, hw, cfg, stats, quant, load_model, retention, n_override, pcfg);
    out["plan_text"] = plan.to_text();
    out["n_batches"] = plan.n_batches;
    cfg.n_batches = plan.n_batches;
    moesim::ActivationTrace trace;
    if (!req.contains("recorded")) {
        trace = moesim::generate_trace(model, cfg, skew, seed);
    } else {
        // Routing recorded by the B200 engine (gate mode): the schedule is
        // rebuilt from the selections the engine actually executed. A
        // decode-only run of S steps is a trace of S single-token steps
        // (prompt_len 1), renumbered by step_offset when printed.
        const json& rj = req["recorded"];
        moesim::BatchGroupConfig tc = cfg;
        tc.prompt_len = rj.value("prompt_len", cfg.prompt_len);
        tc.gen_len = rj.at("gen_len").get<int>();
        trace = moesim::generate_trace(model, tc, moesim::SkewSpec::uniform(), 0);
        const std::vector<std::uint16_t> sel = rj.at("sel").get<std::vector<std::uint16_t>>();
        if (sel.size() != trace.sel.size())
            throw moesim::ConfigError("recorded trace has " + std::to_string(sel.size()) + " ids, expected " +
                                      std::to_string(trace.sel.size()));
        trace.sel = sel;
    }
    out["trace_hash"] = fnv1a(trace.sel.data(), trace.sel.size());
    out["trace_size"] = trace.sel.size();
    if (req.value("want_trace", false)) out["trace"] = trace.sel;

    // Prefetch decisions replayed through the table prefetcher.
    if (req.value("want_prefetch", false)) {
        moesim::PrefetchProvider pp =
            moesim::make_table_prefetcher(table, true, moesim::TendencyAggregation::sum, model.top_k);
        json decisions = json::array();
        for (int s = 0; s < trace.n_steps; ++s)
            for (int l = 0; l < trace.n_layers; ++l) {
                std::span<const std::uint16_t> prev;
                if (l > 0) prev = trace.layer_selections(s, l - 1);
                const moesim::PrefetchDecision d = pp(s, l, prev);
                decisions.push_back({d.expert_ids, d.scores, d.used_fallback});
            }
        out["prefetch"] = decisions;
    }

    moesim::PrefetchProvider provider =
        moesim::make_table_prefetcher(table, true, moesim::TendencyAggregation::sum, model.top_k);
    moesim::ScheduleOptions sopts;
    sopts.immediate_offload = req.value("immediate_offload", true);
    const moesim::Variant v = moesim::variant_from_name(variant);
    const moesim::Schedule sched =
        v == moesim::Variant::klotski
            ? moesim::build_klotski_schedule(plan, trace, provider, sopts)
            : moesim::build_baseline_schedule(v, plan, trace, provider, sopts);
    const moesim::ValidationReport rep = moesim::validate_schedule(sched, trace, plan);
    out["violations"] = rep.violations;
    // "lean": the caller times the reference path (bench.py's simulator CPU
    // baseline) and wants neither the schedule nor the timeline text.
    const bool lean = req.value("lean", false);
    const int off = req.value("step_offset", 0);
    if (!lean && off != 0) {
        moesim::Schedule shifted = sched;
        for (moesim::StreamOp& op : shifted.ops) op.step = static_cast<std::int16_t>(op.step + off);
        out["schedule_text"] = shifted.to_text();
    } else if (!lean) {
        out["schedule_text"] = sched.to_text();
    }
    out["n_ops"] = sched.ops.size();

    if (req.value("simulate", true)) {
        moesim::MemoryLedger ledger =
            moesim::MemoryLedger::for_profile(hw, req.value("enforce_vram", false));
        moesim::SimOptions so;
        so.shared_pcie = req.value("shared_pcie", false);
        try {
            const moesim::SimResult r = moesim::run(sched, plan.cost, plan, ledger, so);
            const moesim::RunMetrics& m = r.metrics;
            out["makespan"] = m.makespan;
            out["compute_busy"] = m.compute_busy;
            out["bubble_time"] = m.bubble_time;
            out["expert_layer_bubble_time"] = m.expert_layer_bubble_time;
            out["throughput_tps"] = m.throughput_tps;
            out["peak_vram"] = m.peak_vram;
            out["participation"] = m.prefetch_participation;
            out["hot_accuracy"] = m.hot_accuracy;
            out["tokens_generated"] = m.tokens_generated;
            const auto& b = m.bubbles;
            out["bubbles"] = {b.startup,      b.intra_attention, b.attn_to_moe, b.intra_gate,
                              b.gate_to_expert, b.intra_expert,  b.moe_to_attn, b.drain};
            if (!lean) {
                out["timeline_csv"] =
                    moesim::timeline_to_string(r.timeline, sched, moesim::TimelineFormat::csv);
                out["timeline_json"] = moesim::timeline_to_string(
                    r.timeline, sched, moesim::TimelineFormat::trace_event_json);
                out["memory_csv"] = moesim::memory_timeline_csv(ledger);
            }
        } catch (const moesim::MemoryInfeasible& e) {
            out["run_error"] = std::string("MemoryInfeasible: ") + e.what();
        } catch (const std::exception& e) {
            out["run_error"] = std::string("error: ") + e.what();
        }
    }
    return out;
}

}  // namespace

extern "C" {

// Returns a malloc'd JSON string; free with parity_free. Errors come back as
// {"error": "..."} (no exception crosses the C boundary).
const char* parity_request(const char* req_json) {
    try {
        return dup(request(req_json).dump());
    } catch (const moesim::MemoryInfeasible& e) {
        return dup(json{{"error", std::string("MemoryInfeasible: ") + e.what()}}.dump());
    } catch (const std::exception& e) {
        return dup(json{{"error", e.what()}}.dump());
    }
}

void parity_free(const char* p) { std::free(const_cast<char*>(p)); }

}  // extern "C"
