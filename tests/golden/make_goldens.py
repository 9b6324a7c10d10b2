"""Regenerate tests/golden/reference_runs.json from the REFERENCE library.

Runs oracle/_ref/libref_parity.so (the unmodified reference sources compiled
by oracle/build_ref.sh, namespace moesim_ref) on a fixed set of requests and
stores its answers: plan text, schedule text, validation, simulated metrics,
timelines and memory CSV (hashed when large). The GPU box has no
/root/reference, so these fixtures carry the reference's behaviour there.

    python tests/golden/make_goldens.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests import parity  # noqa: E402

BIG = ("schedule_text", "timeline_csv", "timeline_json", "memory_csv", "plan_text", "table_text")


def digest(ans):
    out = {}
    for k, v in ans.items():
        if k in BIG and isinstance(v, str) and len(v) > 4000:
            out[k + "_sha256"] = hashlib.sha256(v.encode()).hexdigest()
            out[k + "_len"] = len(v)
        else:
            out[k] = v
    return out


def requests():
    reqs = []
    # toy.cfg-like experiment, every variant, solved n (reference configs/toy.cfg:1-13)
    for v in ("simple", "multibatch_full_prefetch", "strawman_no_reorder", "klotski"):
        reqs.append({"model": {"preset": "toy"}, "hw": {"preset": "toy-hw"},
                     "workload": {"batch_size": 4, "prompt_len": 8, "gen_len": 2}, "skew": {"kind": "zipf", "s": 1.5},
                     "seed": 7, "variant": v, "want_prefetch": True})
    # small fixed-n klotski runs with streamed layers, markov skew, shared PCIe
    reqs.append({"model": {"preset": "toy", "n_layers": 3, "n_experts": 6, "top_k": 2},
                 "hw": {"preset": "toy-hw", "vram_capacity": 40 * 2**20}, "workload": {"batch_size": 3, "prompt_len": 4,
                 "gen_len": 3}, "n": 3, "skew": {"kind": "markov", "s": 1.3, "p": 0.6}, "seed": 11,
                 "shared_pcie": True, "want_prefetch": True, "want_trace": True})
    # Mixtral-8x7B on Env-1 (planner calibration, reference test_planner.cpp:291-309)
    reqs.append({"model": {"preset": "mixtral-8x7b-like"}, "hw": {"preset": "env1"},
                 "workload": {"batch_size": 16, "prompt_len": 512, "gen_len": 2}, "seed": 1, "n": 4,
                 "simulate": True})
    # cfg3-style planner sweep points (n x HBM cap) for Mixtral-8x7B with B200-like rates
    for cap in (16e9, 24e9, 40e9):
        for n in (1, 4, 8):
            reqs.append({"model": {"preset": "mixtral-8x7b-like"},
                         "hw": {"preset": "env2", "vram_capacity": int(cap), "pcie_bandwidth": 55e9,
                                "attn_ps": 500000, "gate_ps": 10000, "expert_ps": 250000},
                         "workload": {"batch_size": 64, "prompt_len": 512, "gen_len": 2}, "seed": 1, "n": n,
                         "streaming_kv": True, "simulate": False})
    return reqs


def main():
    ref = parity.ref()
    out = [{"request": r, "answer": digest(ref(r))} for r in requests()]
    with open(os.path.join(HERE, "reference_runs.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"wrote {len(out)} reference runs")


if __name__ == "__main__":
    main()
