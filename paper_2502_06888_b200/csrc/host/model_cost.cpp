// SPDX-License-Identifier: Apache-2.0
// Model/hardware specs and the affine cost model.
// Semantics follow reference proj/src/model.cpp:6-149 and cost.cpp:11-167.
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "moesim/cost.hpp"
#include "moesim/model.hpp"

namespace moesim {

// ---------------------------------------------------------------- specs ----

void DTypeSpec::validate() const {
    switch (bits_per_element) {
        case 4: case 8: case 16: case 32: return;
        default:
            throw ValidationError("dtype '" + name + "': bits_per_element must be 4, 8, 16 or 32");
    }
}

void ModelSpec::validate() const {
    dtype.validate();
    if (n_layers < 1) throw ValidationError(name + ": n_layers must be >= 1");
    if (top_k < 1) throw ValidationError(name + ": top_k must be >= 1");
    if (top_k > n_experts_per_layer)
        throw ValidationError(name + ": top_k exceeds n_experts_per_layer");
    const bool sizes_ok =
        attention_bytes > 0 && gate_bytes > 0 && expert_bytes > 0 && kv_bytes_per_token > 0;
    if (!sizes_ok) throw ValidationError(name + ": all byte sizes must be > 0");
}

byte_count ModelSpec::layer_bytes() const {
    return attention_bytes + gate_bytes + expert_bytes * static_cast<byte_count>(n_experts_per_layer);
}

byte_count ModelSpec::total_bytes() const { return layer_bytes() * static_cast<byte_count>(n_layers); }

byte_count tensor_bytes(const ModelSpec& spec, TensorKind kind) {
    if (kind == TensorKind::attention) return spec.attention_bytes;
    if (kind == TensorKind::gate) return spec.gate_bytes;
    if (kind == TensorKind::expert) return spec.expert_bytes;
    if (kind == TensorKind::moe_layer)
        return spec.gate_bytes + spec.expert_bytes * static_cast<byte_count>(spec.n_experts_per_layer);
    throw ConfigError("unknown tensor kind");
}

void HardwareProfile::validate() const {
    if (vram_capacity <= 0 || dram_capacity <= 0 || disk_capacity <= 0)
        throw ValidationError(name + ": all capacities must be > 0");
    if (!(pcie_bandwidth > 0.0) || !(disk_bandwidth > 0.0))
        throw ValidationError(name + ": all bandwidths must be > 0");
    if (pinned_bandwidth_factor < 1.0)
        throw ValidationError(name + ": pinned_bandwidth_factor must be >= 1");
    if (transfer_fixed_latency < 0)
        throw ValidationError(name + ": transfer_fixed_latency must be >= 0");
}

namespace {

// A Mixtral-shaped spec: hidden d, ffn f, 8 KV heads of 128 (GQA), bf16.
ModelSpec mixtral_shape(const char* name, int layers, byte_count d, byte_count f) {
    ModelSpec m;
    m.name = name;
    m.n_layers = layers;
    m.n_experts_per_layer = 8;
    m.top_k = 2;
    const byte_count kv_width = 8 * 128;
    m.expert_bytes = 3 * d * f * 2;                        // w1, w3: f x d; w2: d x f
    m.gate_bytes = 8 * d * 2;                              // router: E x d
    m.attention_bytes = (2 * d * d + 2 * d * kv_width) * 2;  // q, o: d x d; k, v: kv x d
    m.kv_bytes_per_token = 2 * kv_width * 2;               // K and V rows, bf16
    m.dtype = {"bf16", 16};
    return m;
}

}  // namespace

ModelSpec mixtral_8x7b_like() { return mixtral_shape("mixtral-8x7b-like", 32, 4096, 14336); }
ModelSpec mixtral_8x22b_like() { return mixtral_shape("mixtral-8x22b-like", 56, 6144, 16384); }

ModelSpec toy_model(int n_layers, int n_experts, int top_k) {
    ModelSpec m;
    m.name = "toy";
    m.n_layers = n_layers;
    m.n_experts_per_layer = n_experts;
    m.top_k = top_k;
    m.expert_bytes = 6 * kMiB;
    m.gate_bytes = 8 * kKiB;
    m.attention_bytes = 2 * kMiB;
    m.kv_bytes_per_token = 512;
    m.dtype = {"bf16", 16};
    return m;
}

HardwareProfile env1_profile() {
    HardwareProfile p;
    p.name = "env1";
    p.vram_capacity = 24'000'000'000;
    p.dram_capacity = 256'000'000'000;
    p.disk_capacity = 2'000'000'000'000;
    p.pcie_bandwidth = 16.75e9;   // ~21 ms per bf16 Mixtral-8x7B expert
    p.pinned_bandwidth_factor = 1.5;
    p.disk_bandwidth = 1.0e9;
    p.attn_compute_per_token = ps_from_us(162.5);  // 2.6 ms at batch 16
    p.gate_compute_per_token = ps_from_us(1.625);
    p.expert_compute_per_token = ps_from_us(900.0);
    p.dequant_ps_per_byte = 0.001;
    return p;
}

HardwareProfile env2_profile() {
    HardwareProfile p;
    p.name = "env2";
    p.vram_capacity = 80'000'000'000;
    p.dram_capacity = 800'000'000'000;
    p.disk_capacity = 1'000'000'000'000;
    p.pcie_bandwidth = 55.0e9;
    p.pinned_bandwidth_factor = 1.5;
    p.disk_bandwidth = 3.0e9;
    p.attn_compute_per_token = ps_from_us(40.0);
    p.gate_compute_per_token = ps_from_us(0.5);
    p.expert_compute_per_token = ps_from_us(220.0);
    p.dequant_ps_per_byte = 0.0005;
    return p;
}

HardwareProfile toy_profile() {
    HardwareProfile p;
    p.name = "toy-hw";
    p.vram_capacity = 64 * kMiB;
    p.dram_capacity = 1 * kGiB;
    p.disk_capacity = 16 * kGiB;
    p.pcie_bandwidth = 4.0e9;
    p.pinned_bandwidth_factor = 1.5;
    p.disk_bandwidth = 0.5e9;
    p.transfer_fixed_latency = ps_from_us(5.0);
    p.attn_compute_per_token = ps_from_us(20.0);
    p.gate_compute_per_token = ps_from_us(0.4);
    p.expert_compute_per_token = ps_from_us(120.0);
    p.dequant_ps_per_byte = 0.001;
    return p;
}

// ----------------------------------------------------------------- cost ----

namespace {

std::int64_t ps_per_byte(double bytes_per_sec) {
    if (bytes_per_sec <= 0.0) throw ConfigError("bandwidth must be > 0");
    return std::llround(1e12 / bytes_per_sec);
}

}  // namespace

std::int64_t route_ps_per_byte(const HardwareProfile& profile, TransferRoute route) {
    switch (route) {
        case TransferRoute::dram_vram_pinned:
        case TransferRoute::vram_dram:
            return ps_per_byte(profile.pcie_bandwidth);
        case TransferRoute::dram_vram_unpinned:
            return ps_per_byte(profile.pcie_bandwidth / profile.pinned_bandwidth_factor);
        case TransferRoute::disk_dram:
            return ps_per_byte(profile.disk_bandwidth);
    }
    throw ConfigError("unknown transfer route");
}

duration_ps transfer_time(const HardwareProfile& profile, byte_count bytes, TransferRoute route) {
    if (bytes < 0) throw ValidationError("transfer_time: negative byte count");
    if (bytes == 0) return profile.transfer_fixed_latency;
    return profile.transfer_fixed_latency + bytes * route_ps_per_byte(profile, route);
}

duration_ps compute_time(const HardwareProfile& profile, LayerKind kind, std::int64_t tokens) {
    if (tokens < 0) throw ValidationError("compute_time: negative token count");
    switch (kind) {
        case LayerKind::attention: return tokens * profile.attn_compute_per_token;
        case LayerKind::gate: return tokens * profile.gate_compute_per_token;
        case LayerKind::expert: return tokens * profile.expert_compute_per_token;
    }
    throw ConfigError("unknown layer kind");
}

duration_ps CostProfile::io_time(byte_count bytes, TransferRoute route) const {
    if (bytes == 0) return transfer_fixed_latency;
    std::int64_t rate = ps_per_byte_pinned;
    if (route == TransferRoute::dram_vram_unpinned) rate = ps_per_byte_unpinned;
    if (route == TransferRoute::disk_dram) rate = ps_per_byte_disk;
    return transfer_fixed_latency + bytes * rate;
}

namespace {

// Memo key: every input that can change the profile (rates rounded the same
// way they enter the integer model).
using MemoKey = std::tuple<std::string, int, int, int, byte_count, byte_count, byte_count,
                           byte_count, std::string, byte_count, byte_count, byte_count,
                           std::int64_t, std::int64_t, std::int64_t, duration_ps, duration_ps,
                           duration_ps, duration_ps, std::int64_t, int, int, int, int>;

struct CostMemo {
    std::mutex mu;
    std::map<MemoKey, CostProfile> entries;
};

CostMemo& memo() {
    static CostMemo m;
    return m;
}

}  // namespace

CostProfile build_cost_profile(const ModelSpec& spec, const HardwareProfile& profile,
                               int batch_size, const std::optional<QuantConfig>& quant) {
    if (batch_size < 1) throw ValidationError("build_cost_profile: batch_size must be >= 1");
    spec.validate();
    profile.validate();
    if (quant) quant->validate();

    const QuantConfig qk = quant ? *quant : QuantConfig{0, 0, 0};
    const MemoKey key{spec.name, spec.n_layers, spec.n_experts_per_layer, spec.top_k,
                      spec.attention_bytes, spec.gate_bytes, spec.expert_bytes,
                      spec.kv_bytes_per_token, profile.name, profile.vram_capacity,
                      profile.dram_capacity, profile.disk_capacity,
                      std::llround(profile.pcie_bandwidth),
                      std::llround(profile.pinned_bandwidth_factor * 1000),
                      std::llround(profile.disk_bandwidth), profile.transfer_fixed_latency,
                      profile.attn_compute_per_token, profile.gate_compute_per_token,
                      profile.expert_compute_per_token,
                      std::llround(profile.dequant_ps_per_byte * 1e6), batch_size, qk.bits,
                      qk.group_size, qk.zero_scale_group_size};
    {
        std::lock_guard<std::mutex> g(memo().mu);
        auto hit = memo().entries.find(key);
        if (hit != memo().entries.end()) return hit->second;
    }

    CostProfile c;
    c.batch_size = batch_size;
    c.top_k = spec.top_k;
    c.n_experts = spec.n_experts_per_layer;
    c.transfer_fixed_latency = profile.transfer_fixed_latency;
    c.ps_per_byte_pinned = route_ps_per_byte(profile, TransferRoute::dram_vram_pinned);
    c.ps_per_byte_unpinned = route_ps_per_byte(profile, TransferRoute::dram_vram_unpinned);
    c.ps_per_byte_disk = route_ps_per_byte(profile, TransferRoute::disk_dram);
    c.kv_bytes_per_token = spec.kv_bytes_per_token;
    c.quantized = quant.has_value();

    // Experts and attention travel quantized when quantization is on; the
    // router is left at native precision.
    const int elem_bytes = spec.dtype.bits_per_element / 8;
    auto on_wire = [&](byte_count native) -> byte_count {
        if (!quant || elem_bytes == 0) return native;
        return quantized_bytes(native / elem_bytes, *quant);
    };
    c.attention_transfer_bytes = on_wire(spec.attention_bytes);
    c.gate_transfer_bytes = spec.gate_bytes;
    c.expert_transfer_bytes = on_wire(spec.expert_bytes);
    c.moe_transfer_bytes = c.gate_transfer_bytes +
                           static_cast<byte_count>(spec.n_experts_per_layer) * c.expert_transfer_bytes;

    c.attn_per_token = profile.attn_compute_per_token;
    c.gate_per_token = profile.gate_compute_per_token;
    c.t_c_e_per_token = profile.expert_compute_per_token;
    if (quant) {
        // Dequant cost spread as if one activated expert serves one batch.
        c.t_c_e_per_token += std::llround(profile.dequant_ps_per_byte *
                                          static_cast<double>(c.expert_transfer_bytes) / batch_size);
    }
    c.t_c_a = c.attn_per_token * batch_size;
    c.t_c_g = c.gate_per_token * batch_size;
    c.t_io_a = c.io_time(c.attention_transfer_bytes, TransferRoute::dram_vram_pinned);
    c.t_io_g = c.io_time(c.gate_transfer_bytes, TransferRoute::dram_vram_pinned);
    c.t_io_e = c.io_time(c.expert_transfer_bytes, TransferRoute::dram_vram_pinned);
    c.t_io_moe = c.io_time(c.moe_transfer_bytes, TransferRoute::dram_vram_pinned);

    std::lock_guard<std::mutex> g(memo().mu);
    memo().entries.emplace(key, c);
    return c;
}

}  // namespace moesim
