#!/usr/bin/env python
"""Headline benchmark: Mixtral-8x7B bf16 decode under a capped HBM budget with
experts streamed from pinned host memory (BASELINE.json configs[1]):
batch 64 x n=8 batch group, 24e9-byte HBM arena, StreamingLLM KV retention
(sink 4 + window 256, the reference's KvRetentionPolicy) so the KV cache stays
in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0. A "step" = one decode step of the whole batch group
(n*bs = 512 tokens) through all 32 layers: attention, router, expert-major
permutation, every active expert's SwiGLU FFN (weights H2D-streamed by the
Klotski schedule), combine, greedy head.
  value : decode tokens/s with the step's inputs already in HBM (device events)
  e2e   : the same through the public C-ABI (kl_engine_step) with host token
          ids in and host next-token ids out, copies inside the timed region
The reference arm (--impl reference) times the CPU port of the same decode
step (oracle/cpu_port.py, C oracle kernels, all host threads) on a bounded
sample: the reference itself (proj/) is a simulator with no numeric path.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s (Mixtral-8x7B, capped HBM)"


T_START = time.perf_counter()


def log(msg):
    """Progress on stderr (the JSON line alone goes to stdout)."""
    print(f"[bench {time.perf_counter() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6650.0), "measured"
    except (OSError, ValueError):
        return 6650.0, "fallback"


def link_peak_gbs(torch, dev):
    """Pinned H2D copy bandwidth of this box (the streaming roofline)."""
    n = 512 * 1024 * 1024
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(6):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return 6 * n / (s.elapsed_time(e) / 1e3) / 1e9


def share_ep_id(rank, world, make_id):
    """Rank 0 creates the NCCL unique id for the engine's EP communicator; all
    ranks receive it over the torch.distributed group (gloo or nccl)."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x, world, device):
    """Max of a host float over ranks (multi-GPU timings: slowest rank)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def engine_config(args, rank, world, ep_id=None):
    gen = 1 + args.warmup + 2 * args.steps
    cfg = {
        "model": {"preset": args.model},
        "workload": {"batch_size": args.batch_size, "n_batches": args.n_batches, "prompt_len": args.prompt_len,
                     "gen_len": gen},
        "hbm_cap_bytes": int(args.hbm_cap),
        "kv_retention": {"mode": "streaming", "sink_tokens": 4, "window_tokens": 256},
        "routing": "gate",
        "prefill": False,
        "record_trace": True,  # the executed routing feeds the reference validator below
        "host_distinct_layers": args.host_distinct_layers,
        "weight_seed": 7 if ep_id is not None else 7 + rank,
    }
    if ep_id is not None:
        cfg["ep"] = {"rank": rank, "world": world, "nccl_id": ep_id}
    if getattr(args, "quant_bits", 0):
        cfg["quant"] = {"bits": args.quant_bits}
    return cfg


def ffn_isolated(torch, dev, D, M, iters=20):
    """The dominant kernel alone, live in this process: the expert FFN
    (kl_expert_ffn, two weight-streaming tcgen05 GEMMs) on the model's expert
    shape with the step's mean routed rows, 8 distinct experts so weights
    come from HBM (> L2), timed back-to-back with CUDA events on the launching
    stream after warm-up; the calls are captured once into a CUDA graph so
    host launch gaps do not count (device time of the kernels)."""
    from paper_2502_06888_b200 import kernels as K
    d, f = D["d"], D["f"]
    ws = [torch.empty(3 * d * f, dtype=torch.bfloat16, device=dev) for _ in range(8)]
    for i, w in enumerate(ws):
        # the engine's expert format: K-blocked W13 [2f, d] and W2 [d, f]
        raw = torch.empty(3 * d * f, dtype=torch.bfloat16, device=dev)
        K.fill_normal(raw, 1000 + i, 0.02)
        w[: 2 * f * d].view(2 * f, d).copy_(K.weights_kblock(raw[: 2 * f * d].view(2 * f, d)))
        w[2 * f * d:].view(d, f).copy_(K.weights_kblock(raw[2 * f * d:].view(d, f)))
        del raw
    xp = torch.empty(max(M, 1) * 8, d, dtype=torch.bfloat16, device=dev)
    K.fill_normal(xp, 999, 1.0)
    y = torch.empty_like(xp)
    h = torch.empty(max(M, 1), f, dtype=torch.bfloat16, device=dev)

    def run(i):
        w = ws[i % 8]
        K.expert_ffn(xp, (i % 8) * M, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h, kblocked=True)
    for i in range(4):
        run(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            run(i)
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    g.replay()
    b.record(st)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / iters * 1e3
    del g
    # The form the engine runs at decode: down-projection splits left as
    # fp32 partials for the block's combine (kl_expert_ffn_kb_deferred).
    us_def = None
    S = K.expert_ffn_deferred_splits(M, d, f)
    if S:
        yp = torch.empty(S, max(M, 1) * 8, d, dtype=torch.float32, device=dev)

        def run_def(i):
            w = ws[i % 8]
            K.expert_ffn_deferred(xp, (i % 8) * M, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), yp,
                                  h, S)
        for i in range(4):
            run_def(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(iters):
                run_def(i)
        g.replay()
        torch.cuda.synchronize()
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        us_def = a.elapsed_time(b) / iters * 1e3
        del g, yp
    byts = 3 * d * f * 2 + M * (2 * d * 2 + 2 * f * 2)
    del ws, xp, y, h
    torch.cuda.empty_cache()
    return us, byts, us_def


def measured_tflops(sustained=False):
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        if key in p:
            return p[key], "measured " + ("sustained" if sustained else "burst")
        return p.get("bf16_tflops", 1590.0), "measured burst"
    except (OSError, ValueError):
        return 1590.0, "fallback"


def prefill_variant(args, link):
    """BASELINE configs[2]: prefill of a batch group (bs 32 x n 8 x 512-token
    prompts = 131,072 tokens) through all layers under the same HBM cap, experts
    streamed; one warm-up pass then one timed pass. Reports prefill tokens/s,
    the pipeline bubble fraction and the expert GEMMs' tensor-pipe rate
    (FLOPs / measured compute time) against the bf16 peak."""
    log('prefill_variant')
    from paper_2502_06888_b200.engine import Engine
    import numpy as np
    bs, n, P = 32, 8, args.prompt_len
    cfg = {"model": {"preset": args.model},
           "workload": {"batch_size": bs, "n_batches": n, "prompt_len": P, "gen_len": 2},
           "hbm_cap_bytes": int(args.hbm_cap),
           "kv_retention": {"mode": "streaming", "sink_tokens": 4, "window_tokens": 256},
           "routing": "gate", "prefill": True, "record_trace": False, "host_distinct_layers": 4}
    eng = Engine(cfg)
    prompt = np.random.default_rng(0).integers(0, eng.info["dims"]["V"], eng.n_seqs * P, dtype=np.int32)
    eng.step(0, prompt)
    eng.reset_log()
    _, ms = eng.step(0, prompt)
    m = eng.report("metrics")
    D = eng.info["dims"]
    flops = 2.0 * 3 * D["d"] * D["f"] * m["expert_rows"]
    t_exp = m["compute_ps_by_kind"]["expert"] * 1e-12
    peak, kind = measured_tflops(sustained=True)  # a seconds-long in-step rate: the sustained peak
    tf = flops / t_exp / 1e12 if t_exp > 0 else 0.0
    out = {"config": f"{args.model} prefill, batch {bs} x n={n} x {P} tokens, HBM cap {args.hbm_cap:.3g} B, "
                     "host copies of the layers aliased onto 4 distinct layers (link bytes unchanged)",
           "value": eng.n_seqs * P / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
           "bubble_fraction": m["bubble_fraction"], "bubbles_ps": m["bubbles_ps"],
           "compute_ms_by_kind": {k: v / 1e9 for k, v in m["compute_ps_by_kind"].items()},
           "h2d_gb_per_step": m["h2d_bytes"] / 1e9, "h2d_frac_of_link_peak": m["h2d_gbs_busy"] / link,
           "expert_gemm_tflops": tf, "tensor_peak_tflops": peak, "tensor_peak_kind": kind,
           "expert_gemm_tensor_frac": tf / peak,
           "resident_expert_layers": eng.info["resident_expert_layers"]}
    eng.close()
    return out


def q4_variant(args, link):
    """Same decode workload with 4-bit streamed experts/attention (Q4T, the
    reference's QuantConfig{4, 64}): the link moves 0.28125x
    the bytes and the dequantisation runs inside the GEMM producer. A second
    engine after the bf16 one is closed; reported beside the headline."""
    log('q4_variant')
    from paper_2502_06888_b200.engine import Engine
    a = argparse.Namespace(**vars(args))
    a.quant_bits = 4
    t0 = time.perf_counter()
    eng = Engine(engine_config(a, 0, 1))
    eng.fill_kv_synthetic(args.prompt_len)
    setup = time.perf_counter() - t0
    step = 1
    for _ in range(args.warmup):
        eng.step(step, None, want_next=False)
        step += 1
    eng.reset_log()
    ms = []
    for _ in range(args.steps):
        _, t = eng.step(step, None, want_next=False)
        ms.append(t)
        step += 1
    m = eng.report("metrics")
    seqs = eng.n_seqs
    n_ops = max(m["expert_ops"], 1)
    D = eng.info["dims"]
    out = {
        "value": args.steps * seqs / (sum(ms) / 1e3), "unit": "tokens/s", "ms_per_step": sum(ms) / args.steps,
        "quant": "Q4T 4-bit, group 64, fp16 scale/zero (reference QuantConfig{4,64})",
        "expert_stream_bytes": eng.info["expert_stream_bytes"],
        "h2d_gb_per_step": m["h2d_bytes"] / args.steps / 1e9, "h2d_gbs_link_busy": m["h2d_gbs_busy"],
        "h2d_frac_of_link_peak": m["h2d_gbs_busy"] / link, "bubble_fraction": m["bubble_fraction"],
        "resident_expert_layers": eng.info["resident_expert_layers"],
        "expert_ffn_us_per_op": m["compute_ps_by_kind"]["expert"] / n_ops / 1e6,
        "expert_ffn_q4_bytes_per_op": eng.info["expert_stream_bytes"] + m["expert_rows"] / n_ops * (2 * D["d"] * 2 + 2 * D["f"] * 2),
        "setup_s": setup,
    }
    eng.close()
    return out


def cpu_baseline(args, warmup=0, repeats=1):
    from oracle import cpu_port
    r = cpu_port.measure(args.model, args.n_batches, args.batch_size, cap=260, repeats=repeats, warmup=warmup)
    return r


def run_reference(args):
    """The reference arm: the CPU path timed on this box's host cores, whole
    decode steps (one batch of the group through all layers per step), so
    steps x ms_per_step is the timed wall time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import cpu_port
    sample = cpu_port.StepSample(args.model, args.batch_size, 260)
    for _ in range(args.warmup):
        sample.decode_step(600)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        sample.decode_step(600)
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = sample.tokens / step_s
    desc = (f"each step: one whole {args.model} decode step of one batch ({args.batch_size} sequences, 260 "
            f"retained KV slots) through all {sample.D['L']} layers (layers aliased onto one layer's weights/KV); "
            f"the group's {args.n_batches} batches are independent steps of this size")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{args.model} decode, batch {args.batch_size} x n={args.n_batches}, CPU port",
                   "batch_size": args.batch_size, "n_batches": args.n_batches},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s_timed": sum(times),
        "note": "reference proj/ is a discrete-event simulator without numerics; its CPU path is the oracle port",
    }
    print(json.dumps(line), flush=True)
    return 0


def simulator_baseline(info, rates, args):
    """Second CPU figure: the reference's own CPU path, the
    discrete-event simulator of oracle/_ref (build_klotski_schedule + run,
    shared-PCIe link) on the cfg2 workload (prompt 512 + generate 128,
    bs 64 x n 8, 24 GB cap) priced with the rates this run measured;
    single-threaded by design. Reports its wall time and simulated tok/s."""
    log('simulator_baseline')
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_parity.so"))
    lib.parity_request.argtypes = [C.c_char_p]
    lib.parity_request.restype = C.c_void_p
    lib.parity_free.argtypes = [C.c_void_p]
    spec = info["spec"]
    gen = 128
    req = {
        "model": {"preset": "toy", "n_layers": spec["n_layers"], "n_experts": spec["n_experts"],
                  "top_k": spec["top_k"], "expert_bytes": spec["expert_bytes"],
                  "attention_bytes": spec["attention_bytes"], "gate_bytes": spec["gate_bytes"],
                  "kv_bytes_per_token": spec["kv_bytes_per_token"]},
        "hw": dict(info["profile"], attn_ps=int(rates["attn_ps_per_token"]), gate_ps=int(rates["gate_ps_per_token"]),
                   expert_ps=int(rates["expert_ps_per_token"]), pcie_bandwidth=float(rates["pcie_bytes_per_s"]),
                   transfer_fixed_latency_ps=0),
        "workload": {"batch_size": args.batch_size, "n_batches": args.n_batches, "prompt_len": args.prompt_len,
                     "gen_len": gen},
        "skew": {"kind": "zipf", "s": 1.5}, "seed": 1, "n": args.n_batches,
        "working_set_override": info["working_set_bytes"], "streaming_kv": info["streaming_kv"],
        "sink_tokens": info["sink_tokens"], "window_tokens": info["window_tokens"],
        "simulate": True, "shared_pcie": True, "lean": True,
    }
    t0 = time.perf_counter()
    ptr = lib.parity_request(json.dumps(req).encode())
    wall = time.perf_counter() - t0
    try:
        out = json.loads(C.string_at(ptr).decode())
    finally:
        lib.parity_free(ptr)
    if "error" in out or "run_error" in out:
        return {"error": out.get("error") or out.get("run_error")}
    toks = args.batch_size * args.n_batches * gen
    mk = out["makespan"] * 1e-12
    return {"kind": "reference", "impl": "oracle/_ref moesim::build_klotski_schedule + moesim::run (shared PCIe)",
            "cores": 1, "nproc": os.cpu_count(), "wall_s": wall, "n_ops": out["n_ops"],
            "value": toks / wall, "unit": "simulated tokens per wall-clock second",
            "simulated_tok_s": out["throughput_tps"], "simulated_makespan_s": mk,
            "simulated_bubble_fraction": out["bubble_time"] / out["makespan"] if out["makespan"] else None,
            "sample": f"prompt {args.prompt_len} + generate {gen}, bs {args.batch_size} x n {args.n_batches}, "
                      f"zipf(1.5) trace, rates measured in this run"}


def decode_engine_run(cfg, warmup, steps, prompt_len):
    """Build an engine, prefill-free decode: warm-up steps, then `steps`
    timed steps (device events per step). Returns (engine, ms list)."""
    from paper_2502_06888_b200.engine import Engine
    cfg = dict(cfg, workload=dict(cfg["workload"], gen_len=1 + warmup + steps))
    eng = Engine(cfg)
    eng.fill_kv_synthetic(prompt_len)
    step = 1
    for _ in range(warmup):
        eng.step(step, None, want_next=False)
        step += 1
    eng.reset_log()
    ms = []
    for _ in range(steps):
        _, t = eng.step(step, None, want_next=False)
        ms.append(t)
        step += 1
    return eng, ms


def resident_variant(args):
    """Compute-exposed decode (the regime of one EP shard that fits HBM, where
    north_star's <10% bubble target applies): the same decode workload with an
    HBM budget (140e9 B) that keeps every expert and attention layer resident,
    so nothing is streamed and the step is the kernels plus the per-layer
    routing round trip. Reports tok/s, the reference bubble fraction and
    breakdown on the measured timeline, and the expert FFN per op."""
    log('resident_variant')
    a = argparse.Namespace(**vars(args))
    a.hbm_cap = 140e9
    steps = max(4, min(args.steps, 20))
    eng, ms = decode_engine_run(engine_config(a, 0, 1), 3, steps, args.prompt_len)
    m = eng.report("metrics")
    val = eng.report("validate")
    D = eng.info["dims"]
    n_ops = max(m["expert_ops"], 1)
    hbm_peak, _ = measured_peaks()
    op_us = m["compute_ps_by_kind"]["expert"] / n_ops / 1e6
    byts = m["expert_bytes"] + m["expert_rows"] / n_ops * (2 * D["d"] * 2 + 2 * D["f"] * 2)
    out = {"config": f"{args.model} bf16 decode, batch {args.batch_size} x n={eng.n_batches}, HBM cap 1.4e11 B "
                     "(all layers resident, nothing streamed)",
           "value": steps * eng.n_seqs / (sum(ms) / 1e3), "unit": "tokens/s", "steps": steps,
           "ms_per_step": sum(ms) / steps, "bubble_fraction": m["bubble_fraction"], "bubbles_ps": m["bubbles_ps"],
           "compute_busy_ms": m["compute_busy_ps"] / 1e9, "makespan_ms": m["makespan_ps"] / 1e9,
           "compute_ms_by_kind": {k: v / 1e9 for k, v in m["compute_ps_by_kind"].items()},
           "resident_expert_layers": eng.info["resident_expert_layers"],
           "resident_attention_layers": eng.info["resident_attention_layers"],
           "h2d_gb_per_step": m["h2d_bytes"] / steps / 1e9,
           "expert_op_us": op_us, "expert_ffn_frac_of_hbm_peak": byts / op_us / 1e3 / hbm_peak,
           "violations": len(val["violations"]), "gpu_launches": m["launches"]}
    eng.close()
    return out


def x22b_variant(args, link):
    """BASELINE configs[3] at N=1: Mixtral-8x22B (56 layers, d 6144, f 16384,
    48q/8kv heads; model.cpp:70-82, 603,979,776 B per expert) bf16 decode,
    batch 64 x n 8, HBM capped at 40e9 B so the experts stream from pinned host
    (the KV of 260 retained positions stays in HBM). The expert-parallel
    streaming-scaling workload of SURVEY 8(e) on one GPU: tok/s, link
    fraction and bubble. Host copies aliased onto 4 distinct layers (link
    bytes unchanged) to bound pinned host memory and setup time."""
    log('x22b_variant')
    a = argparse.Namespace(**vars(args))
    a.model = "mixtral-8x22b"
    a.hbm_cap = 40e9
    a.host_distinct_layers = 4
    steps = 2
    a.steps = steps
    a.warmup = 1
    cfg = engine_config(a, 0, 1)
    # The planner is told the host holds every layer (282 GB of 8x22B host
    # copies; this box's RAM is smaller, hence the aliasing): no disk tier.
    cfg["host_dram_bytes"] = int(1e12)
    t0 = time.perf_counter()
    eng, ms = decode_engine_run(cfg, 1, steps, args.prompt_len)
    m = eng.report("metrics")
    val = eng.report("validate")
    D = eng.info["dims"]
    n_ops = max(m["expert_ops"], 1)
    hbm_peak, _ = measured_peaks()
    op_us = m["compute_ps_by_kind"]["expert"] / n_ops / 1e6
    byts = m["expert_bytes"] + m["expert_rows"] / n_ops * (2 * D["d"] * 2 + 2 * D["f"] * 2)
    h2d = m["h2d_bytes"] / steps
    out = {"config": f"mixtral-8x22b bf16 decode, batch {args.batch_size} x n={eng.n_batches}, HBM cap 4e10 B, "
                     "experts streamed from pinned host (host copies aliased onto 4 distinct layers)",
           "value": steps * eng.n_seqs / (sum(ms) / 1e3), "unit": "tokens/s", "steps": steps,
           "ms_per_step": sum(ms) / steps, "bubble_fraction": m["bubble_fraction"],
           "h2d_gb_per_step": h2d / 1e9, "h2d_gbs_link_busy": m["h2d_gbs_busy"],
           "h2d_frac_of_link_peak": m["h2d_gbs_busy"] / link,
           "link_bound_ceiling_tok_s": eng.n_seqs / (h2d / (link * 1e9)),
           "resident_expert_layers": eng.info["resident_expert_layers"],
           "resident_attention_layers": eng.info["resident_attention_layers"],
           "expert_bytes": m["expert_bytes"], "expert_op_us": op_us,
           "expert_ffn_frac_of_hbm_peak": byts / op_us / 1e3 / hbm_peak,
           "violations": len(val["violations"]), "wall_s": time.perf_counter() - t0}
    eng.close()
    return out


def sweep_variant(args, full=False):
    """BASELINE configs[2]: Mixtral-8x7B prefill 512 + generate 128, swept over
    the batch number n and the HBM cap through the I/O-compute planner
    (the reference's run_sweep, experiment.cpp:342-378, on the engine).
    Stage 1: the engine's per-token rates and the pinned link
    are measured once (kl_measure_profile, decode phase, which dominates a
    128-token generation); stage 2: make_plan solves n and the placement under
    each cap with those rates (a plan_only engine reports solved_n_uncapped
    and the KV-capped n). Each (cap, n) point then runs on the engine: the
    prefill pass (step 0) and two decode steps, timed on the device; the
    group's tok/s is the reference definition bs*n*gen_len / makespan
    (simulator.cpp:264-267) with makespan = prefill + 127 x mean decode step
    (sink 4 + window 256 retention: every decode step sees the same 260
    positions, so the steps are alike). batch 32; host copies aliased onto 4
    distinct layers (link bytes unchanged)."""
    log('sweep_variant')
    from paper_2502_06888_b200.engine import Engine, measure_profile
    import numpy as np
    bs, P, G = 32, args.prompt_len, 128
    caps = (16e9, 24e9, 40e9) if full else (24e9,)
    ns = (1, 2, 4, 8, 12, 16, 24, 32) if full else (2, 8)
    base = {"model": {"preset": args.model},
            "workload": {"batch_size": bs, "n_batches": 8, "prompt_len": P, "gen_len": G},
            "kv_retention": {"mode": "streaming", "sink_tokens": 4, "window_tokens": 256},
            "routing": "gate", "prefill": True, "record_trace": False, "host_distinct_layers": 4}
    prof = measure_profile(dict(base, hbm_cap_bytes=int(24e9)), "decode")
    rates = {"attn_ps": int(prof["attn_ps_per_token"]), "gate_ps": int(prof["gate_ps_per_token"]),
             "expert_ps": int(prof["expert_ps_per_token"]), "pcie_bandwidth": float(prof["pcie_bandwidth"])}
    out = {"config": f"{args.model} prefill {P} + generate {G}, batch {bs}, n x HBM cap grid; host copies aliased onto "
                     "4 distinct layers (link bytes unchanged)",
           "method": "tok/s = bs*n*128 / (prefill_ms + 127 * mean of 2 decode steps), device-timed per step",
           "rates": rates, "caps": {}}
    rng = np.random.default_rng(0)
    for cap in caps:
        key = f"{cap / 1e9:.0f}GB"
        row = {"points": []}
        try:
            pe = Engine(dict(base, hbm_cap_bytes=int(cap), solve_n=True, plan_only=True, **rates))
            row["planner_solved_n"] = pe.info["planner_solved_n"]   # solve_min_n (planner.cpp:58-116)
            row["planner_n"] = pe.info["planner_n"]                 # after the reference KV cap
            row["engine_n"] = pe.info["n_batches"]                  # after the engine's HBM working set
            row["kv_capped"] = pe.info["kv_capped"]
            pe.close()
        except Exception as ex:  # reported, not fatal
            row["planner_error"] = str(ex)[:200]
        grid = sorted(set(ns) | ({row["engine_n"]} if row.get("engine_n") else set()))
        for n in grid:
            pt = {"n": n}
            try:
                cfg = dict(base, hbm_cap_bytes=int(cap), **rates)
                cfg["workload"] = dict(base["workload"], n_batches=n)
                eng = Engine(cfg)
                prompt = rng.integers(0, eng.info["dims"]["V"], eng.n_seqs * P, dtype=np.int32)
                _, pms = eng.step(0, prompt, want_next=False)
                dms = [eng.step(s, None, want_next=False)[1] for s in (1, 2)]
                m = eng.report("metrics")
                dmean = sum(dms) / len(dms)
                makespan_ms = pms + (G - 1) * dmean
                pt.update({"tok_s": bs * n * G / (makespan_ms / 1e3), "prefill_ms": pms, "decode_ms": dmean,
                           "decode_tok_s": bs * n / (dmean / 1e3), "bubble_fraction": m["bubble_fraction"],
                           "resident_expert_layers": eng.info["resident_expert_layers"],
                           "kv_offload": eng.info["kv_offload"]})
                eng.close()
            except Exception as ex:  # infeasible points are reported, not fatal
                pt["error"] = str(ex)[:200]
            row["points"].append(pt)
        ok = [p for p in row["points"] if "tok_s" in p]
        if ok:
            best = max(ok, key=lambda p: p["tok_s"])
            row["measured_best_n"] = best["n"]
            row["measured_best_tok_s"] = best["tok_s"]
            at = [p for p in ok if p["n"] == row.get("engine_n")]
            if at:
                row["solved_n_tok_s"] = at[0]["tok_s"]
                row["solved_over_best"] = at[0]["tok_s"] / best["tok_s"]
        out["caps"][key] = row
    return out


def ablation_variant(args):
    """Table-6-style ablation at the headline scale: the
    reference's schedule variants executed by the engine on the same decode
    workload and HBM cap (experts streamed). simple = row-by-row, one batch
    through every layer reloading its weights (schedule.cpp:636-690);
    multibatch_full_prefetch = whole MoE layers prefetched; strawman_no_reorder
    = split hot/cold without the expert-major reorder; klotski = the headline.
    Host copies of the layers are aliased onto 4 distinct layers to bound setup
    time (link bytes per op are unchanged)."""
    log('ablation_variant')
    out = {}
    for v, steps in (("multibatch_full_prefetch", 2), ("strawman_no_reorder", 2), ("simple", 1)):
        a = argparse.Namespace(**vars(args))
        a.host_distinct_layers = 4
        a.steps = steps
        cfg = engine_config(a, 0, 1)
        cfg["variant"] = v
        cfg["record_trace"] = False
        try:
            t0 = time.perf_counter()
            eng, ms = decode_engine_run(cfg, 1, steps, args.prompt_len)
            m = eng.report("metrics")
            out[v] = {"value": steps * eng.n_seqs / (sum(ms) / 1e3), "unit": "tokens/s",
                      "ms_per_step": sum(ms) / steps, "steps": steps, "bubble_fraction": m["bubble_fraction"],
                      "h2d_gb_per_step": m["h2d_bytes"] / steps / 1e9, "h2d_gbs_link_busy": m["h2d_gbs_busy"],
                      "wall_s": time.perf_counter() - t0}
            eng.close()
        except Exception as ex:  # reported, not fatal
            out[v] = {"error": str(ex)[:300]}
    return out


def run_ours(args):
    import numpy as np
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    from paper_2502_06888_b200.engine import Engine, ep_unique_id

    link = link_peak_gbs(torch, dev)
    t_setup = time.perf_counter()
    use_ep = (world > 1 and args.parallel == "ep") or args.ep1
    ep_id = None
    if use_ep:
        ep_id = share_ep_id(rank, world, ep_unique_id) if world > 1 else ""
    if world > 1 and not use_ep and args.host_distinct_layers == 0:
        args.host_distinct_layers = 4  # replicas: bound pinned host memory per rank
    log('headline engine')
    eng = Engine(engine_config(args, rank, world, ep_id))
    eng.fill_kv_synthetic(args.prompt_len)
    setup_s = time.perf_counter() - t_setup
    seqs = eng.n_seqs
    step = 1
    for _ in range(args.warmup):
        eng.step(step, None, want_next=False)
        step += 1
    eng.reset_log()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    # Timed region 1: inputs resident in HBM (device-fed greedy tokens).
    # (Python's cyclic GC stays off inside both timed regions: a collection
    # pause would land in the end-to-end wall time.)
    import gc
    gc.collect()
    gc.disable()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    dev_ms = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, ms = eng.step(step, None, want_next=False)
        dev_ms.append(ms)
        step += 1
    barrier()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    metrics = eng.report("metrics")
    total_ms = sum(dev_ms)
    # The executed op log through the reference validator (validate_schedule,
    # schedule.cpp:729-860) and the reference ledger replayed on the measured
    # timeline (placement.cpp:257-292), both outside the timed region.
    validation = eng.report("validate")
    ledger = eng.report("ledger")
    # The reference simulator over the executed schedule, priced with this
    # window's measured rates (simulator.cpp:70-287, shared PCIe 99-129).
    simulated = eng.report("simulated")

    # Timed region 2: end to end through the C-ABI with host buffers.
    rng = np.random.default_rng(rank)
    tokens = rng.integers(0, eng.info["dims"]["V"], seqs, dtype=np.int32)
    barrier()
    e2e_ms = []
    t1 = time.perf_counter()
    for _ in range(args.steps):
        tokens, ms = eng.step(step, tokens, want_next=True)
        e2e_ms.append(ms)
        step += 1
    barrier()
    e2e_wall = time.perf_counter() - t1
    gc.enable()

    total_ms = max_over_ranks(total_ms, world, dev)
    e2e_total_ms = max_over_ranks(max(sum(e2e_ms), e2e_wall * 1e3), world, dev)
    value = args.steps * seqs * world / (total_ms / 1e3)
    e2e_value = args.steps * seqs * world / (e2e_total_ms / 1e3)

    # Roofline of the dominant kernel (expert FFN = 2 tcgen05 GEMMs per op):
    # algorithmic bytes per op = expert weights + routed activations in/out.
    D = eng.info["dims"]
    hbm_peak, peak_kind = measured_peaks()
    n_ops = max(metrics["expert_ops"], 1)
    rows = metrics["expert_rows"]
    algo_bytes = n_ops * metrics["expert_bytes"] + rows * (2 * D["d"] * 2 + 2 * D["f"] * 2)
    expert_s = metrics["compute_ps_by_kind"]["expert"] * 1e-12
    achieved = algo_bytes / expert_s / 1e9 if expert_s > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_expert_ffn.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_op")

    info = dict(eng.info)
    n_batches = eng.n_batches
    eng.close()
    eng = None
    prefill = None
    if world == 1 and not args.no_prefill:
        try:
            prefill = prefill_variant(args, link)
        except Exception as ex:  # reported, not fatal
            prefill = {"error": str(ex)[:300]}
    q4 = None
    if world == 1 and not args.no_q4:
        try:
            q4 = q4_variant(args, link)
        except Exception as ex:  # reported, not fatal
            q4 = {"error": str(ex)[:300]}

    resident = ablation = None
    if world == 1 and not args.no_resident:
        try:
            resident = resident_variant(args)
        except Exception as ex:  # reported, not fatal
            resident = {"error": str(ex)[:300]}
    x22b = None
    if world == 1 and not args.no_x22b:
        try:
            x22b = x22b_variant(args, link)
        except Exception as ex:  # reported, not fatal
            x22b = {"error": str(ex)[:300]}
    sweep = None
    if world == 1 and args.sweep != "off":
        try:
            sweep = sweep_variant(args, full=args.sweep == "full")
        except Exception as ex:  # reported, not fatal
            sweep = {"error": str(ex)[:300]}
    if world == 1 and not args.no_ablation:
        ablation = ablation_variant(args)
        ablation["klotski"] = {"value": value, "unit": "tokens/s", "ms_per_step": total_ms / args.steps,
                               "steps": args.steps, "bubble_fraction": metrics["bubble_fraction"],
                               "h2d_gb_per_step": metrics["h2d_bytes"] / args.steps / 1e9,
                               "h2d_gbs_link_busy": metrics["h2d_gbs_busy"], "note": "the headline run"}

    iso = None
    try:
        M = int(round(rows / n_ops))
        us, byts, us_def = ffn_isolated(torch, dev, D, M)
        iso = {"rows": M, "us": us, "achieved_gbs": byts / us / 1e3, "frac": byts / us / 1e3 / hbm_peak,
               "us_deferred_splits": us_def,
               "frac_deferred_splits": byts / us_def / 1e3 / hbm_peak if us_def else None,
               "note": "FFN (owner-fixup form) back-to-back on 8 distinct experts of this shape (HBM-resident "
                       "weights), one CUDA graph of 20 calls timed with events; *_deferred_splits: the form the "
                       "engine runs at decode, whose split reduction is done by the block's combine"}
    except Exception as ex:  # reported, not fatal
        iso = {"error": str(ex)[:200]}

    sim_cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sim_cpu = simulator_baseline(info, simulated["rates"], args)
        except Exception as ex:  # reported, not fatal
            sim_cpu = {"error": str(ex)[:300]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_baseline(args)
            cpu = {"value": r["tok_s"], "unit": "tokens/s", "cores": r["cores"], "kind": "port", "sample": r["sample"]}
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init bf16 weights of the Mixtral-8x7B architecture, random token ids, "
                    "synthetic prefilled KV of 512 positions)",
            "config": {
                "workload": f"{args.model} bf16 decode, batch {args.batch_size} x n={n_batches}, "
                            f"HBM cap {args.hbm_cap:.3g} B, experts streamed from pinned host",
                "model": args.model, "batch_size": args.batch_size, "n_batches": n_batches,
                "prompt_len": args.prompt_len, "kv_retention": "streaming sink 4 + window 256",
                "hbm_cap_bytes": int(args.hbm_cap), "expert_slots": info["expert_slots"],
                "resident_expert_layers": info["resident_expert_layers"],
                "resident_attention_layers": info["resident_attention_layers"],
                "parallelism": (f"ep{world} (expert shards, NCCL all-to-all)" if use_ep else
                                f"replicas x{world}") if world > 1 else "single GPU",
                "l2": "inputs larger than L2 (each step streams the experts of every layer)",
                "host_distinct_layers": args.host_distinct_layers or "all",
            },
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": seqs * 4,
                    "d2h_bytes_per_step": seqs * 4},
            "gpu_launches": metrics["launches"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "expert FFN (tcgen05 SwiGLU GEMM + down GEMM), per compute_expert op; the "
                                   "down projection's k-split partials are summed by the layer block's combine, "
                                   "which runs inside (and is timed with) the block's last compute_expert op",
                         "algorithmic_bytes_per_op": algo_bytes / n_ops,
                         "expert_op_us_in_step": expert_s / n_ops * 1e6,
                         "kernel_isolated": iso},
            "cpu_baseline": cpu,
            "pipeline": {
                "bubble_fraction": metrics["bubble_fraction"],
                "bubbles_ps": metrics["bubbles_ps"],
                "compute_busy_ms": metrics["compute_busy_ps"] / 1e9,
                "makespan_ms": metrics["makespan_ps"] / 1e9,
                "h2d_gb_per_step": metrics["h2d_bytes"] / args.steps / 1e9,
                "h2d_gbs_link_busy": metrics["h2d_gbs_busy"],
                "h2d_gbs_over_makespan": metrics["h2d_gbs_makespan"],
                "link_peak_gbs_measured": link,
                "h2d_frac_of_link_peak": metrics["h2d_gbs_busy"] / link,
                "expert_loads_per_step": metrics["expert_loads"] / args.steps,
                "prefetch_participation": metrics["prefetch_participation"],
                "hot_accuracy": metrics["hot_accuracy"],
                "link_bound_ceiling_tok_s": seqs / (metrics["h2d_bytes"] / args.steps / (link * 1e9)),
            },
            "validate": {"violations": len(validation["violations"]),
                         "first": validation["violations"][:3], "skipped": validation.get("skipped"),
                         "ledger_vram_high_water": ledger["vram_high_water"],
                         "ledger_within_cap": ledger["within_capacity"]},
            "simulated": {"note": "reference moesim::run over the executed schedule with the rates measured in "
                                  "this window (shared PCIe); same window as 'pipeline'",
                          "simulated": {k: simulated["simulated"][k] for k in
                                        ("makespan_ps", "compute_busy_ps", "bubble_fraction", "bubbles_ps")},
                          "measured": {k: simulated["measured"][k] for k in
                                       ("makespan_ps", "compute_busy_ps", "bubble_fraction", "bubbles_ps")},
                          "rates": simulated["rates"]},
            "cpu_baseline_simulator": sim_cpu,
            "resident": resident,
            "ablation": ablation,
            "mixtral_8x22b": x22b,
            "sweep": sweep,
            "setup_s": setup_s,
            "wall_s_timed": wall,
            "q4": q4,
            "prefill": prefill,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="mixtral-8x7b")
    ap.add_argument("--batch-size", type=int, default=64)
    ap.add_argument("--n-batches", type=int, default=8)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--hbm-cap", type=float, default=24e9)
    ap.add_argument("--host-distinct-layers", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-q4", action="store_true", help="skip the 4-bit streamed-expert variant")
    ap.add_argument("--no-prefill", action="store_true", help="skip the prefill (configs[2]) measurement")
    ap.add_argument("--no-resident", action="store_true", help="skip the all-resident (compute-exposed) decode")
    ap.add_argument("--no-x22b", action="store_true", help="skip the Mixtral-8x22B (configs[3]) decode")
    ap.add_argument("--sweep", default="light", choices=["off", "light", "full"],
                    help="configs[2] n x HBM-cap sweep: light = 24 GB cap, n in {2, 8, solved}; "
                         "full = caps {16, 24, 40} GB x n in {1..32} (8 points) + solved n")
    ap.add_argument("--no-ablation", action="store_true", help="skip the schedule-variant ablation")
    ap.add_argument("--quant-bits", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--parallel", default="ep", choices=["ep", "replicas"],
                    help="N>1: expert-parallel shards (default) or independent replicas")
    ap.add_argument("--ep1", action="store_true", help="run the EP engine path even at N=1 (one shard)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
