"""moesim._core (pybind11, the reference's Python module name) drives the
same host pipeline as the C++ API: the schedule text, plan text and simulated
metrics it produces equal the parity driver's answer for the same request
(reference call stack B, experiment.cpp:183-223), and its error types map.
No GPU needed."""
import pytest

from tests import parity


@pytest.fixture(scope="module")
def core():
    import moesim
    import moesim._core as c
    assert c is moesim._core
    return c


def _pipeline(c, variant="klotski", n=3, seed=5):
    spec = c.toy_model(4, 4, 2)
    hw = c.toy_profile()
    cfg = c.BatchGroupConfig(4, n, 8, 3)
    skew = c.SkewSpec.zipf(1.5)
    warm = c.BatchGroupConfig(4, 2, 8, 3)
    wt = c.generate_trace(spec, warm, skew, seed + 1)
    table = c.build_table(wt, spec)
    stats = c.compute_trace_stats(wt, spec.top_k)
    plan = c.make_plan(spec, hw, cfg, stats, n_override=n)
    trace = c.generate_trace(spec, c.BatchGroupConfig(4, plan.n_batches, 8, 3), skew, seed)
    pf = c.make_table_prefetcher(table, True, spec.top_k)
    v = getattr(c.Variant, variant)
    sched = c.build_klotski_schedule(plan, trace, pf) if variant == "klotski" else \
        c.build_baseline_schedule(v, plan, trace, pf)
    return hw, plan, trace, sched


@pytest.mark.parametrize("variant", ["klotski", "strawman_no_reorder", "multibatch_full_prefetch"])
def test_core_matches_parity_driver(core, variant):
    hw, plan, trace, sched = _pipeline(core, variant)
    req = {"hw": {"preset": "toy-hw"}, "model": {"preset": "toy", "n_layers": 4, "n_experts": 4, "top_k": 2},
           "workload": {"batch_size": 4, "prompt_len": 8, "gen_len": 3}, "n": 3,
           "skew": {"kind": "zipf", "s": 1.5}, "seed": 5, "variant": variant, "simulate": True}
    ans = parity.mine()(req)
    assert "error" not in ans, ans
    assert plan.to_text() == ans["plan_text"]
    assert sched.to_text() == ans["schedule_text"]
    assert sched.n_ops == ans["n_ops"]
    assert core.validate_schedule(sched, trace, plan) == ans["violations"]
    m = core.simulate(sched, plan, hw, enforce_vram=False, shared_pcie=False)
    assert m.makespan == ans["makespan"]
    assert m.compute_busy == ans["compute_busy"]
    assert m.bubble_time == ans["bubble_time"]
    assert m.tokens_generated == ans["tokens_generated"]


def test_core_trace_and_presets(core):
    spec = core.mixtral_8x7b_like()
    assert spec.n_experts_per_layer == 8 and spec.top_k == 2
    assert spec.expert_bytes == 3 * 4096 * 14336 * 2
    t = core.generate_trace(core.toy_model(4, 4, 2), core.BatchGroupConfig(2, 2, 4, 2), core.SkewSpec.uniform(), 1)
    sel = t.sel
    assert sel.dtype.name == "uint16" and len(sel) == (2 * 2 * 4 + 1 * 2 * 2) * 4 * 2
    assert core.KvRetentionPolicy.streaming(4, 256).retained(1000) == 260


def test_core_errors_map(core):
    cfg = core.BatchGroupConfig(0, 1, 1, 1)
    with pytest.raises(core.ValidationError):  # reference: batch group fields must be >= 1
        cfg.validate()
    tiny = core.toy_profile()
    tiny.vram_capacity = 1000
    spec = core.toy_model(4, 4, 2)
    warm = core.generate_trace(spec, core.BatchGroupConfig(4, 2, 8, 2), core.SkewSpec.uniform(), 2)
    with pytest.raises(core.MemoryInfeasible):
        core.make_plan(spec, tiny, core.BatchGroupConfig(4, 2, 8, 2), core.compute_trace_stats(warm, 2))
