"""The CPU numeric oracle checked against independent numpy restatements
(no GPU). The oracle is what GPU parity is measured against, so it is pinned
here first: integer paths exactly, floating paths against float64 numpy."""
import numpy as np
import pytest

from tests import oracle_lib as orc


def test_bf16_round_trip_and_rne():
    x = np.array([1.0, -2.5, 3.140625, 1e-3, 65504.0, 1.00390625, 1.01171875], np.float32)
    b = orc.bf16_bits(x)
    back = orc.bits_to_f32(b)
    # round-to-nearest-even on the 16 dropped bits
    ref = ((x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(b, ref)
    assert np.allclose(back, x, rtol=2 ** -8)


def test_normal_fill_is_deterministic_and_unit_variance():
    a = orc.normal_bf16(200001, 99, 1.0)
    assert np.array_equal(a, orc.normal_bf16(200001, 99, 1.0))
    v = orc.bits_to_f32(a)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1.0) < 0.01
    assert np.abs(v).max() <= 2 * np.sqrt(3) + 1e-2  # Irwin-Hall(4) support


@pytest.mark.parametrize("T,k,E", [(1, 1, 1), (100, 2, 8), (513, 6, 64), (7, 8, 8)])
def test_permute_is_a_stable_counting_sort(T, k, E):
    rng = np.random.default_rng(T + E)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    counts, offsets, pos, row_token = orc.permute(idx, E)
    flat = idx.ravel()
    order = np.argsort(flat, kind="stable")
    assert np.array_equal(counts, np.bincount(flat, minlength=E))
    assert np.array_equal(offsets, np.concatenate([[0], np.cumsum(counts)]))
    assert np.array_equal(pos[order], np.arange(T * k))
    assert np.array_equal(row_token, order // k)


def test_gate_topk_matches_float64_and_tie_rule():
    T, d, E, k = 50, 512, 8, 2
    x = orc.normal_bf16(T * d, 1, 1.0).reshape(T, d)
    w = orc.normal_bf16(E * d, 2, 0.05).reshape(E, d)
    logits, idx, wt = orc.gate_topk(x, w, k)
    ref = orc.bits_to_f32(x).astype(np.float64) @ orc.bits_to_f32(w).astype(np.float64).T
    assert np.abs(logits - ref).max() < 1e-4
    top = np.argsort(-ref, axis=1, kind="stable")[:, :k]
    margin = np.sort(ref, axis=1)[:, -k] - np.sort(ref, axis=1)[:, -k - 1]
    sure = margin > 1e-3
    assert np.array_equal(idx[sure], top[sure])
    sel = np.take_along_axis(ref, top, 1)
    p = np.exp(sel - sel[:, :1])
    p /= p.sum(1, keepdims=True)
    assert np.abs(wt[sure] - p[sure]).max() < 1e-5
    # identical rows tie -> lowest ids
    _, idx2, w2 = orc.gate_topk(x, np.tile(w[:1], (E, 1)), k)
    assert (idx2 == np.array([0, 1])).all() and np.allclose(w2, 0.5)


def test_combine_and_ffn_against_float64():
    T, k, d, f = 9, 2, 256, 512
    R = T * k
    y = orc.normal_bf16(R * d, 5, 1.0).reshape(R, d)
    pos = np.random.default_rng(1).permutation(R).astype(np.int32)
    w = np.random.default_rng(2).random((T, k)).astype(np.float32)
    resid = orc.normal_bf16(T * d, 6, 1.0).reshape(T, d)
    out = orc.bits_to_f32(orc.combine(y, pos, w, resid))
    yf = orc.bits_to_f32(y).astype(np.float64)
    ref = orc.bits_to_f32(resid) + (w[:, :, None] * yf[pos.reshape(T, k)]).sum(1)
    assert np.abs(out - ref).max() <= 2 ** -7 * np.abs(ref).max()
    x = orc.normal_bf16(5 * d, 7, 1.0).reshape(5, d)
    w13 = orc.normal_bf16(2 * f * d, 8, 0.05).reshape(2 * f, d)
    w2 = orc.normal_bf16(d * f, 9, 0.05).reshape(d, f)
    got = orc.bits_to_f32(orc.expert_ffn(x, w13, w2))
    xf, a, b = (orc.bits_to_f32(t).astype(np.float64) for t in (x, w13, w2))
    g, u = xf @ a[:f].T, xf @ a[f:].T
    hh = orc.bits_to_f32(orc.bf16_bits((g / (1 + np.exp(-g)) * u).astype(np.float32))).astype(np.float64)
    ref = hh @ b.T
    assert np.abs(got - ref).max() <= 1e-2 * np.abs(ref).max()


def test_coactivation_counts_match_the_reference_rule():
    # update_table semantics (reference correlation.cpp:123-140): every (a, b)
    # pair of one token increments; layer 0 increments the marginal.
    E, k, T = 6, 2, 40
    rng = np.random.default_rng(3)
    prev = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    cur = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    table = np.zeros(2 * E * E, np.int64)
    marg = np.zeros(E, np.int64)
    orc.coact_update(prev, cur, E, 2, table, marg)
    orc.coact_update(prev, cur, E, 0, table, marg)
    ref = np.zeros((E, E), np.int64)
    for t in range(T):
        for a in prev[t]:
            for b in cur[t]:
                ref[a, b] += 1
    assert np.array_equal(table[E * E:].reshape(E, E), ref)
    assert np.array_equal(marg, np.bincount(cur.ravel(), minlength=E))
    hist = np.bincount(prev.ravel(), minlength=E).astype(np.int32)
    assert np.array_equal(orc.predict_scores(hist, table, E, 2), hist @ ref)


def test_decode_attention_against_float64():
    Hq, Hkv, hd, cap, sink, n = 4, 2, 64, 12, 2, 3
    kc = orc.normal_bf16(n * cap * Hkv * hd, 1, 1.0)
    vc = orc.normal_bf16(n * cap * Hkv * hd, 2, 1.0)
    q = orc.normal_bf16(n * Hq * hd, 3, 1.0).reshape(n, Hq * hd)
    pos = np.array([3, 11, 40], np.int32)
    seq = np.arange(n, dtype=np.int32)
    out = orc.bits_to_f32(orc.attn_decode(q, Hq * hd, pos, seq, Hq, Hkv, hd, kc, vc, cap, hd ** -0.5))
    K = orc.bits_to_f32(kc).reshape(n, cap, Hkv, hd).astype(np.float64)
    V = orc.bits_to_f32(vc).reshape(n, cap, Hkv, hd).astype(np.float64)
    Q = orc.bits_to_f32(q).reshape(n, Hq, hd).astype(np.float64)
    for t in range(n):
        m = min(pos[t] + 1, cap)
        for h in range(Hq):
            s = K[t, :m, h // 2] @ Q[t, h] * hd ** -0.5
            p = np.exp(s - s.max())
            ref = (p / p.sum()) @ V[t, :m, h // 2]
            assert np.abs(out[t].reshape(Hq, hd)[h] - ref).max() < 2e-2
