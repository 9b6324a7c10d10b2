// SPDX-License-Identifier: Apache-2.0
// moesim._core — Python bindings of the host API (replaces the reference's
// one-line stub, proj/bindings/py_module.cpp:1-2; module name and package as
// in proj/CMakeLists.txt:28-37). The same library (libklotski.so) also holds
// the B200 engine and kernels; this module exposes the planner / schedule /
// simulator / trace surface so Python callers can plan, build and price a
// Klotski schedule exactly as the C++ API does, and feed measured B200 rates
// back into make_plan. Exceptions map to Python exceptions (MemoryInfeasible
// keeps its deficits).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "moesim/error.hpp"
#include "moesim/experiment.hpp"
#include "moesim/model.hpp"
#include "moesim/planner.hpp"
#include "moesim/quant.hpp"
#include "moesim/schedule.hpp"
#include "moesim/simulator.hpp"
#include "moesim/trace.hpp"

namespace py = pybind11;
using namespace moesim;

namespace {

// Opaque holder: the plugin point (schedule.hpp:113-114) crosses Python as a
// handle, so a table prefetcher keeps its C++ state (online updates) intact.
struct Prefetcher {
    PrefetchProvider fn;
};

py::dict bubbles_dict(const BubbleBreakdown& b) {
    py::dict d;
    d["startup"] = b.startup;
    d["intra_attention"] = b.intra_attention;
    d["attn_to_moe"] = b.attn_to_moe;
    d["intra_gate"] = b.intra_gate;
    d["gate_to_expert"] = b.gate_to_expert;
    d["intra_expert"] = b.intra_expert;
    d["moe_to_attn"] = b.moe_to_attn;
    d["drain"] = b.drain;
    return d;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "moesim host API (Klotski planner, schedule, simulator) backed by the B200 build";

    // Exception types mirror moesim/error.hpp (error.hpp:11-49).
    static py::exception<ConfigError> config_exc(m, "ConfigError", PyExc_ValueError);
    static py::exception<ValidationError> validation_exc(m, "ValidationError", PyExc_ValueError);
    static py::exception<ParseError> parse_exc(m, "ParseError", PyExc_ValueError);
    static py::exception<AccountingError> accounting_exc(m, "AccountingError", PyExc_RuntimeError);
    static py::exception<MemoryInfeasible> mem_exc(m, "MemoryInfeasible", PyExc_MemoryError);
    py::register_exception_translator([](std::exception_ptr p) {
        try {
            if (p) std::rethrow_exception(p);
        } catch (const MemoryInfeasible& e) {
            py::set_error(mem_exc, e.what());
        } catch (const ConfigError& e) {
            py::set_error(config_exc, e.what());
        } catch (const ValidationError& e) {
            py::set_error(validation_exc, e.what());
        } catch (const ParseError& e) {
            py::set_error(parse_exc, e.what());
        } catch (const AccountingError& e) {
            py::set_error(accounting_exc, e.what());
        }
    });

    py::class_<ModelSpec>(m, "ModelSpec")
        .def(py::init<>())
        .def_readwrite("name", &ModelSpec::name)
        .def_readwrite("n_layers", &ModelSpec::n_layers)
        .def_readwrite("n_experts_per_layer", &ModelSpec::n_experts_per_layer)
        .def_readwrite("top_k", &ModelSpec::top_k)
        .def_readwrite("attention_bytes", &ModelSpec::attention_bytes)
        .def_readwrite("gate_bytes", &ModelSpec::gate_bytes)
        .def_readwrite("expert_bytes", &ModelSpec::expert_bytes)
        .def_readwrite("kv_bytes_per_token", &ModelSpec::kv_bytes_per_token)
        .def("validate", &ModelSpec::validate)
        .def("layer_bytes", &ModelSpec::layer_bytes)
        .def("total_bytes", &ModelSpec::total_bytes);
    m.def("mixtral_8x7b_like", &mixtral_8x7b_like);
    m.def("mixtral_8x22b_like", &mixtral_8x22b_like);
    m.def("toy_model", &toy_model, py::arg("n_layers") = 4, py::arg("n_experts") = 4, py::arg("top_k") = 2);

    py::class_<HardwareProfile>(m, "HardwareProfile")
        .def(py::init<>())
        .def_readwrite("name", &HardwareProfile::name)
        .def_readwrite("vram_capacity", &HardwareProfile::vram_capacity)
        .def_readwrite("dram_capacity", &HardwareProfile::dram_capacity)
        .def_readwrite("disk_capacity", &HardwareProfile::disk_capacity)
        .def_readwrite("pcie_bandwidth", &HardwareProfile::pcie_bandwidth)
        .def_readwrite("pinned_bandwidth_factor", &HardwareProfile::pinned_bandwidth_factor)
        .def_readwrite("disk_bandwidth", &HardwareProfile::disk_bandwidth)
        .def_readwrite("transfer_fixed_latency", &HardwareProfile::transfer_fixed_latency)
        .def_readwrite("attn_compute_per_token", &HardwareProfile::attn_compute_per_token)
        .def_readwrite("gate_compute_per_token", &HardwareProfile::gate_compute_per_token)
        .def_readwrite("expert_compute_per_token", &HardwareProfile::expert_compute_per_token)
        .def_readwrite("dequant_ps_per_byte", &HardwareProfile::dequant_ps_per_byte)
        .def("validate", &HardwareProfile::validate);
    m.def("env1_profile", &env1_profile);
    m.def("env2_profile", &env2_profile);
    m.def("toy_profile", &toy_profile);

    py::class_<BatchGroupConfig>(m, "BatchGroupConfig")
        .def(py::init<>())
        .def(py::init([](int bs, int n, int prompt, int gen) {
                 BatchGroupConfig c;
                 c.batch_size = bs;
                 c.n_batches = n;
                 c.prompt_len = prompt;
                 c.gen_len = gen;
                 return c;
             }),
             py::arg("batch_size"), py::arg("n_batches"), py::arg("prompt_len"), py::arg("gen_len"))
        .def_readwrite("batch_size", &BatchGroupConfig::batch_size)
        .def_readwrite("n_batches", &BatchGroupConfig::n_batches)
        .def_readwrite("prompt_len", &BatchGroupConfig::prompt_len)
        .def_readwrite("gen_len", &BatchGroupConfig::gen_len)
        .def("generated_tokens", &BatchGroupConfig::generated_tokens)
        .def("validate", &BatchGroupConfig::validate);

    py::class_<KvRetentionPolicy> kv(m, "KvRetentionPolicy");
    py::enum_<KvRetentionPolicy::Mode>(kv, "Mode")
        .value("full", KvRetentionPolicy::Mode::full)
        .value("streaming", KvRetentionPolicy::Mode::streaming);
    kv.def(py::init<>())
        .def_static("streaming", [](int sink, int window) {
            KvRetentionPolicy p;
            p.mode = KvRetentionPolicy::Mode::streaming;
            p.sink_tokens = sink;
            p.window_tokens = window;
            return p;
        }, py::arg("sink_tokens") = 4, py::arg("window_tokens") = 256)
        .def_readwrite("mode", &KvRetentionPolicy::mode)
        .def_readwrite("sink_tokens", &KvRetentionPolicy::sink_tokens)
        .def_readwrite("window_tokens", &KvRetentionPolicy::window_tokens)
        .def("retained", &KvRetentionPolicy::retained);

    py::class_<SkewSpec>(m, "SkewSpec")
        .def_static("uniform", &SkewSpec::uniform)
        .def_static("zipf", &SkewSpec::zipf)
        .def_static("markov", &SkewSpec::markov)
        .def("__str__", &SkewSpec::to_string);

    py::class_<QuantConfig>(m, "QuantConfig")
        .def(py::init<>())
        .def_readwrite("bits", &QuantConfig::bits)
        .def_readwrite("group_size", &QuantConfig::group_size)
        .def_readwrite("zero_scale_group_size", &QuantConfig::zero_scale_group_size);
    m.def("quantized_bytes", &quantized_bytes);
    m.def("fit_minmax",
          [](py::array_t<float, py::array::c_style | py::array::forcecast> g, int bits) {
              const QuantParams p = fit_minmax(std::span<const float>(g.data(), static_cast<size_t>(g.size())), bits);
              return py::make_tuple(p.scale, p.zero);
          },
          py::arg("group"), py::arg("bits") = 4);
    m.def("dequantize",
          [](py::array_t<std::uint8_t, py::array::c_style> packed, py::array_t<std::uint16_t, py::array::c_style> scales,
             py::array_t<std::uint16_t, py::array::c_style> zeros, std::size_t n_elements, int bits, int group) {
              QuantizedTensor q;
              q.cfg.bits = bits;
              q.cfg.group_size = group;
              q.n_elements = n_elements;
              q.packed.assign(packed.data(), packed.data() + packed.size());
              q.scales_f16.assign(scales.data(), scales.data() + scales.size());
              q.zeros_f16.assign(zeros.data(), zeros.data() + zeros.size());
              const std::vector<float> v = dequantize(q);
              return py::array_t<float>(static_cast<py::ssize_t>(v.size()), v.data());
          },
          py::arg("packed"), py::arg("scales_f16"), py::arg("zeros_f16"), py::arg("n_elements"), py::arg("bits") = 4,
          py::arg("group_size") = 64,
          "moesim::dequantize of a QuantizedTensor (flat little-endian code stream, per-group fp16 params)");

    py::class_<ActivationTrace>(m, "ActivationTrace")
        .def_readonly("n_steps", &ActivationTrace::n_steps)
        .def_readonly("n_layers", &ActivationTrace::n_layers)
        .def_readonly("n_batches", &ActivationTrace::n_batches)
        .def_readonly("batch_size", &ActivationTrace::batch_size)
        .def_readonly("top_k", &ActivationTrace::top_k)
        .def_readonly("n_experts", &ActivationTrace::n_experts)
        .def_property_readonly("sel", [](const ActivationTrace& t) {
            return py::array_t<std::uint16_t>(static_cast<py::ssize_t>(t.sel.size()), t.sel.data());
        })
        .def("offset", &ActivationTrace::offset)
        .def("to_string", [](const ActivationTrace& t) { return trace_to_string(t); });
    m.def("generate_trace", &generate_trace, py::arg("spec"), py::arg("cfg"), py::arg("skew"), py::arg("seed"));
    m.def("load_trace", &load_trace);
    py::class_<TraceStats>(m, "TraceStats");
    m.def("compute_trace_stats", &compute_trace_stats);

    py::class_<CorrelationTable>(m, "CorrelationTable");
    m.def("build_table", &build_table);

    py::enum_<ExpertLoadModel>(m, "ExpertLoadModel")
        .value("best", ExpertLoadModel::best)
        .value("measured", ExpertLoadModel::measured)
        .value("worst", ExpertLoadModel::worst);
    py::class_<PlacementConfig>(m, "PlacementConfig")
        .def(py::init<>())
        .def_readwrite("working_set_override", &PlacementConfig::working_set_override)
        .def_readwrite("window_reserve_layers", &PlacementConfig::window_reserve_layers)
        .def_readwrite("inflight_cold_experts", &PlacementConfig::inflight_cold_experts);
    py::class_<PipelinePlan>(m, "PipelinePlan")
        .def_readonly("n_batches", &PipelinePlan::n_batches)
        .def_readonly("K", &PipelinePlan::K)
        .def_readonly("batch_size", &PipelinePlan::batch_size)
        .def_readonly("kv_capped", &PipelinePlan::kv_capped)
        .def_readonly("solved_n_uncapped", &PipelinePlan::solved_n_uncapped)
        .def_readonly("warnings", &PipelinePlan::warnings)
        .def_property_readonly("resident_expert_layers", [](const PipelinePlan& p) {
            int r = 0;
            for (Tier t : p.placement.expert_tier) r += t == Tier::vram;
            return r;
        })
        .def_property_readonly("kv_in_vram", [](const PipelinePlan& p) { return p.placement.kv_tier == Tier::vram; })
        .def_property_readonly("working_set_bytes", [](const PipelinePlan& p) { return p.placement.working_set_bytes; })
        .def("to_text", &PipelinePlan::to_text);
    m.def("make_plan", &make_plan, py::arg("spec"), py::arg("profile"), py::arg("cfg"), py::arg("stats"),
          py::arg("quant") = std::nullopt, py::arg("model") = ExpertLoadModel::measured,
          py::arg("retention") = KvRetentionPolicy{}, py::arg("n_override") = std::nullopt,
          py::arg("pcfg") = PlacementConfig{});

    py::enum_<Variant>(m, "Variant")
        .value("simple", Variant::simple)
        .value("multibatch_full_prefetch", Variant::multibatch_full_prefetch)
        .value("strawman_no_reorder", Variant::strawman_no_reorder)
        .value("klotski", Variant::klotski);
    py::class_<Schedule>(m, "Schedule")
        .def_property_readonly("n_ops", [](const Schedule& s) { return s.ops.size(); })
        .def("to_text", &Schedule::to_text);
    py::class_<Prefetcher>(m, "PrefetchProvider");
    m.def("make_table_prefetcher",
          [](const CorrelationTable& table, bool online_update, int top_k) {
              return Prefetcher{make_table_prefetcher(table, online_update, TendencyAggregation::sum, top_k)};
          },
          py::arg("table"), py::arg("online_update") = true, py::arg("top_k") = 1);
    m.def("build_klotski_schedule", [](const PipelinePlan& plan, const ActivationTrace& trace, const Prefetcher& pf) {
        return build_klotski_schedule(plan, trace, pf.fn);
    });
    m.def("build_baseline_schedule",
          [](Variant v, const PipelinePlan& plan, const ActivationTrace& trace, const Prefetcher* pf) {
              return build_baseline_schedule(v, plan, trace, pf ? pf->fn : PrefetchProvider{});
          },
          py::arg("variant"), py::arg("plan"), py::arg("trace"), py::arg("prefetch") = nullptr);
    m.def("validate_schedule", [](const Schedule& s, const ActivationTrace& t, const PipelinePlan& p) {
        return validate_schedule(s, t, p).violations;
    });

    py::class_<RunMetrics>(m, "RunMetrics")
        .def_readonly("makespan", &RunMetrics::makespan)
        .def_readonly("compute_busy", &RunMetrics::compute_busy)
        .def_readonly("bubble_time", &RunMetrics::bubble_time)
        .def_readonly("expert_layer_bubble_time", &RunMetrics::expert_layer_bubble_time)
        .def_readonly("throughput_tps", &RunMetrics::throughput_tps)
        .def_readonly("peak_vram", &RunMetrics::peak_vram)
        .def_readonly("prefetch_participation", &RunMetrics::prefetch_participation)
        .def_readonly("hot_accuracy", &RunMetrics::hot_accuracy)
        .def_readonly("tokens_generated", &RunMetrics::tokens_generated)
        .def_property_readonly("bubbles", [](const RunMetrics& r) { return bubbles_dict(r.bubbles); })
        .def_property_readonly("bubble_fraction", [](const RunMetrics& r) {
            return r.makespan > 0 ? static_cast<double>(r.bubble_time) / r.makespan : 0.0;
        });
    m.def("simulate",
          [](const Schedule& s, const PipelinePlan& plan, const HardwareProfile& hw, bool enforce_vram,
             bool shared_pcie) {
              MemoryLedger ledger = MemoryLedger::for_profile(hw, enforce_vram);
              SimOptions o;
              o.shared_pcie = shared_pcie;
              return run(s, plan.cost, plan, ledger, o).metrics;
          },
          py::arg("schedule"), py::arg("plan"), py::arg("profile"), py::arg("enforce_vram") = false,
          py::arg("shared_pcie") = true,
          "moesim::run with a ledger for the profile; returns RunMetrics");

    py::class_<ExperimentConfig>(m, "ExperimentConfig")
        .def(py::init<>())
        .def_readwrite("model", &ExperimentConfig::model)
        .def_readwrite("hardware", &ExperimentConfig::hardware)
        .def_readwrite("workload", &ExperimentConfig::workload)
        .def_readwrite("skew", &ExperimentConfig::skew)
        .def_readwrite("seed", &ExperimentConfig::seed)
        .def_readwrite("n_override", &ExperimentConfig::n_override)
        .def_readwrite("variants", &ExperimentConfig::variants)
        .def_readwrite("quant", &ExperimentConfig::quant)
        .def_readwrite("kv_retention", &ExperimentConfig::kv_retention)
        .def_readwrite("load_model", &ExperimentConfig::load_model)
        .def_readwrite("sweep_n", &ExperimentConfig::sweep_n)
        .def_readwrite("shared_pcie", &ExperimentConfig::shared_pcie)
        .def_readwrite("output_dir", &ExperimentConfig::output_dir)
        .def_readwrite("export_timelines", &ExperimentConfig::export_timelines);
    m.def("load_experiment_config", &load_experiment_config);
    m.def("simulate_variant",
          [](const ExperimentConfig& cfg, Variant v, std::optional<int> n) {
              SingleRun r = simulate_variant(cfg, v, n);
              return py::make_tuple(r.plan, r.metrics);
          },
          py::arg("cfg"), py::arg("variant") = Variant::klotski, py::arg("n_override") = std::nullopt);
    m.def("run_sweep", [](const ExperimentConfig& cfg) {
        SweepResult r = run_sweep(cfg);
        py::list pts;
        for (const SweepPoint& p : r.points) pts.append(py::make_tuple(p.n, p.batch_size, p.metrics));
        return py::make_tuple(r.solved_n, pts);
    });
    m.def("metrics_to_json", &metrics_to_json);
}
