"""BASELINE configs[4]: DeepSeek-V2-Lite-shaped fine-grained MoE (64 routed
experts top-6 + 2 shared experts of 1408, GQA attention in place of MLA)
decode under a capped HBM budget, in gate mode and in trace-replay mode with
markov-skewed routing (stresses the permutation and the correlation-aware
prefetcher). python tools/deepseek_run.py [--cap 12e9] [--steps 3]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200.engine import Engine  # noqa: E402


def run(routing, cap, steps, bs, n):
    cfg = {"model": {"preset": "deepseek-v2-lite"},
           "workload": {"batch_size": bs, "n_batches": n, "prompt_len": 512, "gen_len": 2 + steps},
           "hbm_cap_bytes": int(cap), "kv_retention": {"mode": "streaming", "sink_tokens": 4, "window_tokens": 256},
           "routing": routing, "prefill": False, "record_trace": routing == "replay",
           "skew": {"kind": "markov", "s": 1.5, "p": 0.8}, "trace_seed": 5}
    eng = Engine(cfg)
    eng.fill_kv_synthetic(512)
    eng.step(1, None, want_next=False)
    eng.reset_log()
    ms = [eng.step(2 + s, None, want_next=False)[1] for s in range(steps)]
    m = eng.report("metrics")
    out = {"routing": routing, "tok_s": steps * eng.n_seqs / (sum(ms) / 1e3), "ms_per_step": float(np.mean(ms)),
           "bubble_fraction": m["bubble_fraction"], "prefetch_participation": m["prefetch_participation"],
           "hot_accuracy": m["hot_accuracy"], "expert_loads_per_step": m["expert_loads"] / steps,
           "h2d_gb_per_step": m["h2d_bytes"] / steps / 1e9, "h2d_gbs_busy": m["h2d_gbs_busy"],
           "resident_expert_layers": eng.info["resident_expert_layers"],
           "compute_ms_by_kind": {k: v / 1e9 / steps for k, v in m["compute_ps_by_kind"].items()}}
    if routing == "replay":
        v = eng.report("validate")["violations"]
        out["violations"] = len(v)
        out["violation_examples"] = v[:3]
    eng.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap", type=float, default=12e9)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--bs", type=int, default=64)
    ap.add_argument("--n", type=int, default=8)
    a = ap.parse_args()
    res = {"config": f"deepseek-v2-lite (64 routed top-6 + 2 shared), bs {a.bs} x n {a.n}, cap {a.cap:.3g} B",
           "gate": run("gate", a.cap, a.steps, a.bs, a.n), "replay_markov": run("replay", a.cap, a.steps, a.bs, a.n)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
