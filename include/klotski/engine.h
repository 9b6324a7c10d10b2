/* SPDX-License-Identifier: Apache-2.0
 *
 * klotski/engine.h — C-ABI of the B200 execution engine: the drop-in
 * replacement for the reference's simulated execution of a Klotski schedule.
 *
 * Reference interfaces this replaces / drives:
 *   moesim::run(const Schedule&, const CostProfile&, const PipelinePlan&,
 *               MemoryLedger&, const SimOptions&)      proj/include/moesim/simulator.hpp:66-67
 *   moesim::build_klotski_schedule(plan, trace, prefetch, opts)
 *                                                      proj/include/moesim/schedule.hpp:126-128
 *   moesim::make_table_prefetcher / PrefetchProvider   proj/include/moesim/schedule.hpp:113-120
 *   moesim::make_plan                                  proj/include/moesim/planner.hpp:73-79
 *   moesim::simulate_variant (binding entry)           proj/include/moesim/experiment.hpp:76-77
 *
 * The engine plans with moesim::make_plan, then for every (step, layer)
 * emits the reference's Algorithm-1 ops online (same StreamOp log as
 * build_klotski_schedule for the same routing) and executes each op on
 * B200: copies on dedicated CUDA streams from pinned host memory into a
 * bounded expert-slot pool, sm_100a kernels on the compute stream,
 * dependencies as cudaEvents. Routing comes from the gate kernel (mode
 * "gate") or is forced from a moesim::generate_trace trace ("replay"). The
 * measured timeline is reported with the reference's RunMetrics /
 * bubble_stats definitions.
 *
 * Conventions: opaque handle; 0 = success, non-zero = failure with the
 * message available from kl_engine_last_error(). The code names the moesim
 * exception class the C++ layer raised (reference error.hpp:11-49, plus
 * DeviceError for CUDA / NCCL / OS failures), see KL_E* below; strings returned through
 * `char**` are malloc'd and released with kl_engine_free_string(). Host
 * buffers are plain pointers. Not thread-safe per handle.
 *
 * Config JSON keys (all optional unless noted):
 *   model: {preset: "mixtral-8x7b"|"mixtral-8x22b"|"tiny"|"deepseek-v2-lite",
 *           n_layers, d, f, heads, kv_heads, head_dim, experts, top_k, vocab,
 *           rope_theta, norm_eps, score_mode}
 *   workload: {batch_size, n_batches, prompt_len, gen_len}
 *   hbm_cap_bytes, host_dram_bytes, pcie_bandwidth, attn_ps, gate_ps, expert_ps
 *   kv_retention: {mode: "full"|"streaming", sink_tokens, window_tokens}
 *   variant: "klotski"|"strawman_no_reorder"|"multibatch_full_prefetch"|"simple"
 *   routing: "gate"|"replay";  skew: {kind, s, p};  trace_seed, warmup_seed
 *   weight_seed, host_distinct_layers (0 = every layer distinct)
 *   expert_slots (0 = auto), ffn_chunk_rows, record_trace, record_hidden
 *   ep: {rank, world, backend: "nccl"|"loopback", nccl_id, group}  expert-parallel
 *       shard (experts e with e % world == rank); loopback = G engines of one
 *       process on one device (host threads), rendezvous by group name
 *   profile: {measure: "decode"|"prefill"}  plan with rates measured here
 *   solve_n: true  let make_plan solve n (ignores workload.n_batches)
 *   plan_only: true  plan and stop (kl_engine_describe only: n, solved_n_uncapped,
 *                    placement, working set; no memory is allocated, steps fail)
 */
#ifndef KLOTSKI_ENGINE_H
#define KLOTSKI_ENGINE_H

#include <stdint.h>

/* Return codes of every kl_engine_* / kl_measure_profile entry point. */
#define KL_OK 0
#define KL_EOTHER 1         /* any other std::exception */
#define KL_EMEMORY 2        /* moesim::MemoryInfeasible (model + workload do not fit) */
#define KL_ECONFIG 3        /* moesim::ConfigError */
#define KL_EVALIDATION 4    /* moesim::ValidationError */
#define KL_EPARSE 5         /* moesim::ParseError */
#define KL_ERANGE 6         /* moesim::RangeError */
#define KL_EACCOUNTING 7    /* moesim::AccountingError (ledger / scheduler invariant) */
#define KL_EDEVICE 8        /* moesim::DeviceError (CUDA / NCCL / OS) */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kl_engine kl_engine;

int kl_engine_create(const char* config_json, kl_engine** out);
void kl_engine_destroy(kl_engine* e);
const char* kl_engine_last_error(const kl_engine* e);
void kl_engine_free_string(char* s);

/* Plan / placement / arena layout as JSON (plan_text = PipelinePlan::to_text). */
int kl_engine_describe(kl_engine* e, char** json_out);

/* Fill every layer's KV cache with synthetic values for positions
 * [0, positions) of every sequence (stands in for a prefill so decode steps
 * can be measured alone). */
int kl_engine_fill_kv_synthetic(kl_engine* e, int positions, uint64_t seed);

/* Run one step of the batch group through all layers. step 0 is the prefill
 * (tokens_in: n_batches*batch_size*prompt_len ids, sequence-major), steps
 * >= 1 decode one token per sequence (n_batches*batch_size ids). tokens_in
 * NULL = feed the previous step's greedy tokens (device resident).
 * next_tokens_out (host, n_batches*batch_size) may be NULL.
 * step_ms_out (may be NULL) receives the device time of the whole step. */
int kl_engine_step(kl_engine* e, int step, const int32_t* tokens_in, int32_t* next_tokens_out,
                   double* step_ms_out);

/* Report of everything executed since create (or the last reset):
 * what = "metrics" | "schedule" | "timeline_csv" | "timeline_json" |
 *        "prefetch" | "trace" | "stats" | "validate" | "hidden" */
int kl_engine_report(kl_engine* e, const char* what, char** json_out);

/* Forget the executed op log and timeline (weights, KV and tables stay). */
int kl_engine_reset_log(kl_engine* e);

/* Expert parallelism: rank 0 creates an NCCL unique id (256 hex chars +
 * NUL into hex_out[257]) and shares it; every rank then passes it as
 * config "ep": {"rank": r, "world": G, "nccl_id": hex}. 0 = success. */
int kl_ep_unique_id(char* hex_out);

/* Planner stage 1 ("measure, then solve"): time this
 * engine's kernels on the config's model shapes (attention block, router,
 * expert FFN at the phase's mean routed rows) and the pinned H2D link on one
 * and two copy streams. phase = "decode" | "prefill". JSON out: per-token
 * ps rates for moesim::HardwareProfile (model.hpp:43-58:
 * attn/gate/expert_compute_per_token) and pcie_bandwidth (bytes/s). Feeds
 * moesim::build_cost_profile (cost.cpp:106-167) and make_plan
 * (planner.cpp:167-239); config key "profile": {"measure": phase} makes
 * kl_engine_create plan with it. Errors: kl_engine_last_error(NULL). */
int kl_measure_profile(const char* config_json, const char* phase, char** json_out);

/* Copy the group's current hidden states [T, d] (bf16 bits) to host. */
int kl_engine_read_hidden(kl_engine* e, uint16_t* host, int64_t n_elems);

#ifdef __cplusplus
}
#endif

#endif /* KLOTSKI_ENGINE_H */
