"""Host-layer parity (no GPU): this repo's moesim implementation against the
reference, on the same requests.

1. Committed reference answers (tests/golden/reference_runs.json, generated
   from oracle/_ref by tests/golden/make_goldens.py) — runs anywhere.
2. Live differential runs against oracle/_ref/libref_parity.so on randomised
   workloads (schedules, prefetch decisions, simulated timelines, ledgers,
   planner output) — runs where the reference library was built.
3. The reference's own 100 unit test cases compiled against this repo
   (needs /root/reference; the oracle pin is the same sources against the
   reference library).
"""
import json
import os
import subprocess

import numpy as np
import pytest

from tests import parity
from tests.golden.make_goldens import digest

ROOT = parity.ROOT
REF_TESTS = "/root/reference/proj/tests"


def test_committed_reference_runs_match():
    with open(os.path.join(ROOT, "tests", "golden", "reference_runs.json")) as f:
        runs = json.load(f)
    mine = parity.mine()
    for run in runs:
        got = digest(mine(run["request"]))
        assert got == run["answer"], run["request"]


def _random_request(rng):
    E = int(rng.choice([2, 4, 6, 8]))
    k = int(rng.integers(1, min(E, 3) + 1))
    layers = int(rng.integers(1, 5))
    skew = [{"kind": "uniform"}, {"kind": "zipf", "s": float(rng.uniform(0.5, 2.0))},
            {"kind": "markov", "s": 1.5, "p": float(rng.uniform(0, 1))}][int(rng.integers(0, 3))]
    req = {
        "model": {"preset": "toy", "n_layers": layers, "n_experts": E, "top_k": k},
        "hw": {"preset": "toy-hw", "vram_capacity": int(rng.choice([20, 28, 40, 64, 256])) * 2**20},
        "workload": {"batch_size": int(rng.integers(1, 6)), "prompt_len": int(rng.integers(1, 6)),
                     "gen_len": int(rng.integers(1, 4))},
        "skew": skew,
        "seed": int(rng.integers(1, 1000)),
        "variant": str(rng.choice(["simple", "multibatch_full_prefetch", "strawman_no_reorder", "klotski"])),
        "shared_pcie": bool(rng.integers(0, 2)),
        "immediate_offload": bool(rng.integers(0, 2)),
        "enforce_vram": bool(rng.integers(0, 2)),
        "streaming_kv": bool(rng.integers(0, 2)),
        "want_prefetch": True,
        "want_trace": True,
    }
    if rng.integers(0, 3):
        req["n"] = int(rng.integers(1, 6))
    if rng.integers(0, 4) == 0:
        req["quant"] = True
    return req


@pytest.mark.skipif(not os.path.exists(parity.REF_LIB), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(60))
def test_random_workloads_match_reference(seed):
    rng = np.random.default_rng(seed)
    req = _random_request(rng)
    assert parity.mine()(req) == parity.ref()(req), req


@pytest.mark.skipif(not os.path.exists(parity.REF_LIB), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("preset,hw", [("mixtral-8x7b-like", "env1"), ("mixtral-8x22b-like", "env2"),
                                       ("mixtral-8x7b-like", "env2")])
def test_planner_presets_match_reference(preset, hw):
    for bs in (4, 16, 64):
        req = {"model": {"preset": preset}, "hw": {"preset": hw},
               "workload": {"batch_size": bs, "prompt_len": 512, "gen_len": 2}, "seed": 3, "simulate": False}
        assert parity.mine()(req) == parity.ref()(req)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference test sources not present")
def test_reference_unit_tests_pass_against_this_repo():
    subprocess.run(["make", "-C", ROOT, "build/mine_unit_tests"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(ROOT, "build", "mine_unit_tests")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "failed: 0; checks:" in r.stdout and "test cases: 100" in r.stdout, r.stdout


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")),
                    reason="oracle/_ref not built")
def test_oracle_is_pinned_by_reference_tests():
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "test cases: 100, failed: 0" in r.stdout, r.stdout + r.stderr[-2000:]
