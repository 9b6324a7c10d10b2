// SPDX-License-Identifier: Apache-2.0
// Discrete-event pricing of a schedule, metrics, bubble attribution and
// timeline/memory exports. Semantics: reference proj/src/simulator.cpp
// (op_duration 13-33, run 70-287, bubble_stats 289-326, throughput 328-331,
// exports 333-396). The B200 executor (engine/) reuses finalize_metrics()
// and bubble_stats() on measured timestamps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <queue>
#include <sstream>

#include "metrics.hpp"
#include "moesim/simulator.hpp"

namespace moesim {

namespace {

duration_ps priced(const StreamOp& op, const CostProfile& cost) {
    switch (op.kind) {
        case OpKind::compute_attention: return op.token_count * cost.attn_per_token;
        case OpKind::compute_gate: return op.token_count * cost.gate_per_token;
        case OpKind::compute_expert: return op.token_count * cost.t_c_e_per_token;
        case OpKind::offload_expert:
        case OpKind::offload_weights: return 0;  // dropping read-only weights moves no bytes
        case OpKind::window_stage:
            return op.payload_bytes == 0 ? 0 : cost.io_time(op.payload_bytes, TransferRoute::disk_dram);
        default: return cost.io_time(op.payload_bytes, op.route);
    }
}

bool rides_pcie(StreamId s) {
    return s == StreamId::weight_load || s == StreamId::expert_load || s == StreamId::cache_load ||
           s == StreamId::cache_store;
}

std::string deadlock_report(const Schedule& s, const std::vector<char>& done) {
    std::ostringstream os;
    os << "simulator deadlock; unfinished ops:";
    int shown = 0;
    for (const StreamOp& op : s.ops) {
        if (done[op.id]) continue;
        if (shown++ >= 8) {
            os << " ...";
            break;
        }
        os << " " << op.id << "(" << op_kind_name(op.kind) << " waits on";
        for (std::int32_t d : op.deps)
            if (!done[d]) os << ' ' << d;
        os << ")";
    }
    return os.str();
}

// Event-driven engine state. Streams are unit-capacity FIFOs; the optional
// shared-PCIe mode splits the link evenly among in-flight transfers.
class Sim {
  public:
    Sim(const Schedule& s, const CostProfile& c, const SimOptions& o)
        : s_(s), cost_(c), opts_(o), n_(s.ops.size()) {
        start_.assign(n_, -1);
        end_.assign(n_, -1);
        started_.assign(n_, 0);
        done_.assign(n_, 0);
        waiting_on_.assign(n_, 0);
        dependents_.resize(n_);
        left_.assign(n_, 0.0);
        version_.assign(n_, 0);
        for (const StreamOp& op : s.ops) {
            waiting_on_[op.id] = static_cast<int>(op.deps.size());
            for (std::int32_t d : op.deps) dependents_[d].push_back(op.id);
        }
    }

    void execute() {
        start_ready();
        std::size_t finished = 0;
        while (finished < n_) {
            if (queue_.empty()) throw AccountingError(deadlock_report(s_, done_));
            const Ev ev = queue_.top();
            queue_.pop();
            if (ev.version != version_[ev.op] || done_[ev.op]) continue;
            const StreamOp& op = s_.ops[ev.op];
            if (opts_.shared_pcie && rides_pcie(op.stream) && end_[ev.op] < 0) {
                refresh_link(ev.time);
                if (left_[ev.op] > 0.5) continue;  // superseded by a reschedule
                end_[ev.op] = ev.time;
                link_.erase(std::find(link_.begin(), link_.end(), ev.op));
                refresh_link(ev.time);
            }
            done_[ev.op] = 1;
            ++finished;
            const int st = static_cast<int>(op.stream);
            busy_[st] = false;
            free_at_[st] = end_[ev.op];
            note_effects(op, LedgerEffect::When::at_end, end_[ev.op]);
            for (std::int32_t w : dependents_[ev.op]) --waiting_on_[w];
            start_ready();
        }
    }

    void replay_ledger(const PipelinePlan& plan, MemoryLedger& ledger) const {
        const ModelSpec& m = plan.model;
        ledger.alloc(plan.placement.activation_tier,
                     m.kv_bytes_per_token * static_cast<byte_count>(s_.batch_size) * s_.n_batches,
                     "activations", 0);
        for (int j = 0; j < plan.placement.n_layers; ++j) {
            if (plan.placement.expert_tier[j] == Tier::vram)
                ledger.alloc(Tier::vram, m.expert_bytes * m.n_experts_per_layer, "res:e:" + std::to_string(j), 0);
            if (plan.placement.gate_tier[j] == Tier::vram)
                ledger.alloc(Tier::vram, m.gate_bytes, "res:g:" + std::to_string(j), 0);
            if (plan.placement.attention_tier[j] == Tier::vram)
                ledger.alloc(Tier::vram, m.attention_bytes, "res:a:" + std::to_string(j), 0);
        }
        std::vector<Effect> ordered = effects_;
        std::stable_sort(ordered.begin(), ordered.end(), [](const Effect& a, const Effect& b) {
            if (a.time != b.time) return a.time < b.time;
            if (a.is_alloc != b.is_alloc) return !a.is_alloc;  // frees first at equal time
            return a.seq < b.seq;
        });
        for (const Effect& e : ordered) {
            if (e.is_alloc) ledger.alloc(e.tier, e.bytes, *e.tag, e.time);
            else ledger.free(*e.tag, e.time);
        }
    }

    std::vector<SimEvent> timeline() const {
        std::vector<SimEvent> t;
        t.reserve(n_);
        for (const StreamOp& op : s_.ops)
            t.push_back({op.id, op.stream, start_[op.id], end_[op.id], op.payload_bytes, op.token_count});
        return t;
    }

  private:
    struct Ev {
        duration_ps time;
        std::int64_t seq;
        std::int32_t op;
        int version;
        bool operator>(const Ev& o) const { return time != o.time ? time > o.time : seq > o.seq; }
    };
    struct Effect {
        duration_ps time;
        bool is_alloc;
        Tier tier;
        byte_count bytes;
        std::int32_t seq;
        const std::string* tag;
    };

    void post(duration_ps t, std::int32_t op) {
        ++version_[op];
        queue_.push({t, seq_++, op, version_[op]});
    }

    void note_effects(const StreamOp& op, LedgerEffect::When when, duration_ps t) {
        for (const LedgerEffect& e : op.ledger)
            if (e.when == when) effects_.push_back({t, e.is_alloc, e.tier, e.bytes, op.id, &e.tag});
    }

    // Fluid link: drain everyone's remaining work for the elapsed time at the
    // current share, then re-post completion events at the new share.
    void refresh_link(duration_ps now) {
        const int m = static_cast<int>(link_.size());
        if (m == 0) {
            link_clock_ = now;
            return;
        }
        const double elapsed = static_cast<double>(now - link_clock_);
        for (std::int32_t id : link_) left_[id] = std::max(0.0, left_[id] - elapsed / m);
        link_clock_ = now;
        for (std::int32_t id : link_) post(now + static_cast<duration_ps>(std::ceil(left_[id] * m)), id);
    }

    void begin(std::int32_t id) {
        const StreamOp& op = s_.ops[id];
        const int st = static_cast<int>(op.stream);
        duration_ps t0 = free_at_[st];
        for (std::int32_t d : op.deps) t0 = std::max(t0, end_[d]);
        t0 = std::max<duration_ps>(t0, 0);
        const duration_ps dur = priced(op, cost_);
        start_[id] = t0;
        started_[id] = 1;
        busy_[st] = true;
        note_effects(op, LedgerEffect::When::at_start, t0);
        if (opts_.shared_pcie && rides_pcie(op.stream) && dur > 0) {
            refresh_link(t0);
            left_[id] = static_cast<double>(dur);
            link_.push_back(id);
            refresh_link(t0);
        } else {
            end_[id] = t0 + dur;
            post(t0 + dur, id);
        }
    }

    // One attempt on stream st: FIFO head when its deps are met; inside a
    // reorder group, the member with the earliest dependency-ready time
    // (ties: lower expert id).
    bool try_stream(int st) {
        if (busy_[st]) return false;
        const auto& order = s_.streams[st];
        std::size_t& head = next_[st];
        while (head < order.size() && started_[order[head]]) ++head;
        if (head >= order.size()) return false;
        const StreamOp& h = s_.ops[order[head]];
        if (h.reorder_group < 0) {
            if (waiting_on_[h.id] > 0) return false;
            begin(h.id);
            return true;
        }
        std::int32_t pick = -1;
        duration_ps pick_ready = 0;
        for (std::size_t i = head; i < order.size(); ++i) {
            const StreamOp& c = s_.ops[order[i]];
            if (c.reorder_group != h.reorder_group) break;
            if (started_[c.id] || waiting_on_[c.id] > 0) continue;
            duration_ps ready = 0;
            for (std::int32_t d : c.deps) ready = std::max(ready, end_[d]);
            const bool better = pick < 0 || ready < pick_ready ||
                                (ready == pick_ready && c.expert < s_.ops[pick].expert);
            if (better) {
                pick = c.id;
                pick_ready = ready;
            }
        }
        if (pick < 0) return false;
        begin(pick);
        return true;
    }

    void start_ready() {
        for (bool moved = true; moved;) {
            moved = false;
            for (int st = 0; st < kNumStreams; ++st) moved |= try_stream(st);
        }
    }

    const Schedule& s_;
    const CostProfile& cost_;
    SimOptions opts_;
    std::size_t n_;
    std::vector<duration_ps> start_, end_;
    std::vector<char> started_, done_;
    std::vector<int> waiting_on_;
    std::vector<std::vector<std::int32_t>> dependents_;
    std::array<std::size_t, kNumStreams> next_{};
    std::array<duration_ps, kNumStreams> free_at_{};
    std::array<bool, kNumStreams> busy_{};
    std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> queue_;
    std::int64_t seq_ = 0;
    std::vector<double> left_;
    std::vector<int> version_;
    std::vector<std::int32_t> link_;
    duration_ps link_clock_ = 0;
    std::vector<Effect> effects_;
};

}  // namespace

namespace detail {

std::int64_t replay_ledger_on_timeline(const Schedule& schedule, std::span<const SimEvent> timeline,
                                       const PipelinePlan& plan, MemoryLedger& ledger) {
    struct Eff {
        duration_ps time;
        bool is_alloc;
        Tier tier;
        byte_count bytes;
        std::int64_t seq;
        const std::string* tag;
    };
    std::vector<Eff> effs;
    std::int64_t seq = 0;
    for (const SimEvent& ev : timeline) {
        const StreamOp& op = schedule.ops[ev.op_id];
        for (const LedgerEffect& e : op.ledger)
            effs.push_back({e.when == LedgerEffect::When::at_start ? ev.start : ev.end, e.is_alloc, e.tier, e.bytes,
                            seq++, &e.tag});
    }
    const ModelSpec& m = plan.model;
    ledger.alloc(plan.placement.activation_tier,
                 m.kv_bytes_per_token * static_cast<byte_count>(schedule.batch_size) * schedule.n_batches, "activations",
                 0);
    for (int j = 0; j < plan.placement.n_layers; ++j) {
        if (plan.placement.expert_tier[j] == Tier::vram)
            ledger.alloc(Tier::vram, m.expert_bytes * m.n_experts_per_layer, "res:e:" + std::to_string(j), 0);
        if (plan.placement.gate_tier[j] == Tier::vram)
            ledger.alloc(Tier::vram, m.gate_bytes, "res:g:" + std::to_string(j), 0);
        if (plan.placement.attention_tier[j] == Tier::vram)
            ledger.alloc(Tier::vram, m.attention_bytes, "res:a:" + std::to_string(j), 0);
    }
    std::stable_sort(effs.begin(), effs.end(), [](const Eff& a, const Eff& b) {
        if (a.time != b.time) return a.time < b.time;
        if (a.is_alloc != b.is_alloc) return !a.is_alloc;
        return a.seq < b.seq;
    });
    std::int64_t carried = 0;
    for (const Eff& e : effs) {
        if (e.is_alloc) {
            if (ledger.live(*e.tag)) ledger.free(*e.tag, e.time);  // re-allocation of a carried-in tag
            ledger.alloc(e.tier, e.bytes, *e.tag, e.time);
        } else if (ledger.live(*e.tag)) {
            ledger.free(*e.tag, e.time);
        } else {
            ++carried;
        }
    }
    return carried;
}

void finalize_metrics(const Schedule& schedule, std::span<const SimEvent> timeline,
                      byte_count peak_vram, RunMetrics& m) {
    m = RunMetrics{};
    for (const SimEvent& e : timeline) {
        m.makespan = std::max(m.makespan, e.end);
        if (e.stream == StreamId::compute) m.compute_busy += e.end - e.start;
    }
    m.bubble_time = m.makespan - m.compute_busy;
    m.bubbles = bubble_stats(timeline, schedule);
    m.expert_layer_bubble_time = m.bubbles.gate_to_expert + m.bubbles.intra_expert;
    m.peak_vram = peak_vram;
    m.tokens_generated = static_cast<std::int64_t>(schedule.batch_size) * schedule.n_batches * schedule.n_steps;
    m.throughput_tps = m.makespan > 0 ? static_cast<double>(m.tokens_generated) / sec_from_ps(m.makespan) : 0.0;
    if (!schedule.prefetch_records.empty()) {
        double part = 0.0, acc = 0.0;
        for (const LayerPrefetchRecord& r : schedule.prefetch_records) {
            int hits = 0, top_hits = 0;
            for (int e : r.prefetched) {
                hits += std::find(r.activated.begin(), r.activated.end(), e) != r.activated.end();
                top_hits += std::find(r.hottest.begin(), r.hottest.end(), e) != r.hottest.end();
            }
            const int k = static_cast<int>(std::max<std::size_t>(1, r.prefetched.size()));
            part += static_cast<double>(hits) / k;
            acc += static_cast<double>(top_hits) / k;
        }
        m.prefetch_participation = part / schedule.prefetch_records.size();
        m.hot_accuracy = acc / schedule.prefetch_records.size();
    }
}

}  // namespace detail

SimResult run(const Schedule& schedule, const CostProfile& cost, const PipelinePlan& plan,
              MemoryLedger& ledger, const SimOptions& opts) {
    Sim sim(schedule, cost, opts);
    sim.execute();
    sim.replay_ledger(plan, ledger);
    SimResult r;
    r.timeline = sim.timeline();
    detail::finalize_metrics(schedule, r.timeline, ledger.high_water(Tier::vram), r.metrics);
    return r;
}

BubbleBreakdown bubble_stats(std::span<const SimEvent> timeline, const Schedule& schedule) {
    BubbleBreakdown b;
    std::vector<const SimEvent*> cs;
    duration_ps makespan = 0;
    for (const SimEvent& e : timeline) {
        makespan = std::max(makespan, e.end);
        if (e.stream == StreamId::compute) cs.push_back(&e);
    }
    if (cs.empty()) return b;
    std::sort(cs.begin(), cs.end(), [](const SimEvent* x, const SimEvent* y) { return x->start < y->start; });
    b.startup = cs.front()->start;
    b.drain = makespan - cs.back()->end;
    for (std::size_t i = 1; i < cs.size(); ++i) {
        const duration_ps gap = cs[i]->start - cs[i - 1]->end;
        if (gap <= 0) continue;
        const Phase p = schedule.ops[cs[i - 1]->op_id].phase;
        const Phase q = schedule.ops[cs[i]->op_id].phase;
        using P = Phase;
        if (p == P::attention && q == P::attention) b.intra_attention += gap;
        else if (p == P::attention && (q == P::gate || q == P::expert)) b.attn_to_moe += gap;
        else if (p == P::gate && q == P::gate) b.intra_gate += gap;
        else if (p == P::gate && q == P::expert) b.gate_to_expert += gap;
        else if (p == P::expert && q == P::expert) b.intra_expert += gap;
        else b.moe_to_attn += gap;
    }
    return b;
}

double throughput(const RunMetrics& metrics, const BatchGroupConfig& cfg) {
    if (metrics.makespan <= 0) return 0.0;
    return static_cast<double>(cfg.generated_tokens()) / sec_from_ps(metrics.makespan);
}

namespace {

std::string micros(duration_ps ps) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%lld.%06lld", static_cast<long long>(ps / kPsPerUs),
                  static_cast<long long>(ps % kPsPerUs));
    return buf;
}

}  // namespace

std::string timeline_to_string(std::span<const SimEvent> timeline, const Schedule& schedule,
                               TimelineFormat format) {
    std::ostringstream os;
    if (format == TimelineFormat::csv) {
        os << "op,stream,kind,step,layer,batch,expert,start_ps,end_ps,bytes,tokens\n";
        for (const SimEvent& e : timeline) {
            const StreamOp& op = schedule.ops[e.op_id];
            os << e.op_id << ',' << stream_name(e.stream) << ',' << op_kind_name(op.kind) << ','
               << op.step << ',' << op.layer << ',' << op.batch << ',' << op.expert << ',' << e.start
               << ',' << e.end << ',' << e.bytes << ',' << e.tokens << "\n";
        }
        return os.str();
    }
    os << "{\"displayTimeUnit\":\"ms\",\"traceEvents\":[";
    for (std::size_t i = 0; i < timeline.size(); ++i) {
        const SimEvent& e = timeline[i];
        const StreamOp& op = schedule.ops[e.op_id];
        if (i) os << ',';
        os << "{\"name\":\"" << op_kind_name(op.kind) << " s" << op.step << " l" << op.layer;
        if (op.batch >= 0) os << " b" << op.batch;
        if (op.expert >= 0) os << " e" << op.expert;
        os << "\",\"cat\":\"" << stream_name(e.stream) << "\",\"ph\":\"X\",\"ts\":" << micros(e.start)
           << ",\"dur\":" << micros(e.end - e.start) << ",\"pid\":0,\"tid\":" << static_cast<int>(e.stream)
           << ",\"args\":{\"op\":" << e.op_id << ",\"bytes\":" << e.bytes << ",\"tokens\":" << e.tokens
           << "}}";
    }
    os << "]}\n";
    return os.str();
}

void export_timeline(std::span<const SimEvent> timeline, const Schedule& schedule,
                     const std::string& path, TimelineFormat format) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw ParseError("export_timeline: cannot open '" + path + "' for writing");
    f << timeline_to_string(timeline, schedule, format);
    if (!f) throw ParseError("export_timeline: write to '" + path + "' failed");
}

std::string memory_timeline_csv(const MemoryLedger& ledger) {
    std::ostringstream os;
    os << "time_ps,vram_bytes,dram_bytes,disk_bytes,event,tag\n";
    byte_count occ[4] = {0, 0, 0, 0};
    for (const MemoryLedger::Event& e : ledger.events()) {
        occ[static_cast<int>(e.tier)] += e.is_alloc ? e.bytes : -e.bytes;
        os << e.time << ',' << occ[0] << ',' << occ[1] + occ[2] << ',' << occ[3] << ','
           << (e.is_alloc ? "alloc" : "free") << ',' << e.tag << "\n";
    }
    return os.str();
}

}  // namespace moesim
