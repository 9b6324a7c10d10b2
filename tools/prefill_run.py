"""Prefill measurement (BASELINE configs[2] shape): one batch group's prompt
(bs x n sequences x prompt_len tokens) through all layers with experts
streamed under the HBM cap; repeated step-0 passes are timed.
python tools/prefill_run.py [--bs 8] [--n 8] [--prompt 512] [--reps 2]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral-8x7b")
    ap.add_argument("--bs", type=int, default=8)
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--hbm-cap", type=float, default=24e9)
    a = ap.parse_args()
    cfg = {"model": {"preset": a.model},
           "workload": {"batch_size": a.bs, "n_batches": a.n, "prompt_len": a.prompt, "gen_len": 2},
           "hbm_cap_bytes": int(a.hbm_cap),
           "kv_retention": {"mode": "streaming", "sink_tokens": 4, "window_tokens": 256},
           "routing": "gate", "prefill": True, "record_trace": False, "host_distinct_layers": 4}
    t0 = time.time()
    eng = Engine(cfg)
    setup = time.time() - t0
    rng = np.random.default_rng(0)
    V = eng.info["dims"]["V"]
    prompt = rng.integers(0, V, eng.n_seqs * a.prompt, dtype=np.int32)
    eng.step(0, prompt)  # warm-up
    eng.reset_log()
    ms = []
    for _ in range(a.reps):
        _, t = eng.step(0, prompt)
        ms.append(t)
    m = eng.report("metrics")
    toks = eng.n_seqs * a.prompt
    out = {"prefill_tokens_per_step": toks, "ms_per_step": ms, "tok_s": toks / (np.median(ms) / 1e3),
           "bubble_fraction": m["bubble_fraction"], "bubbles_ps": m["bubbles_ps"],
           "compute_ms_by_kind": {k: v / 1e9 / a.reps for k, v in m["compute_ps_by_kind"].items()},
           "h2d_gb_per_step": m["h2d_bytes"] / a.reps / 1e9, "h2d_gbs_busy": m["h2d_gbs_busy"],
           "resident_expert_layers": eng.info["resident_expert_layers"], "setup_s": setup}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
