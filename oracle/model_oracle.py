"""CPU model oracle for the engine's numerics (TEST INFRASTRUCTURE).

Regenerates the engine's synthetic weights bit-exactly (same SplitMix64
tensor seeds as csrc/engine/engine.cpp, same Irwin-Hall stream as
kl_fill_normal_bf16) and runs one decoder layer at a time with the C oracle
kernels: RMSNorm, QKV GEMM, RoPE + KV append, prefill/decode attention,
O projection + residual, router, expert-major permutation, SwiGLU experts,
combine. Used teacher-forced: each layer starts from the GPU's own input
hidden state (and optionally the GPU's routing), so per-layer differences are
the kernels' rounding, not accumulated drift.
"""
import numpy as np

from oracle import pyoracle as orc

M64 = (1 << 64) - 1
KIND_EXPERT, KIND_ATTN, KIND_GATE, KIND_EMBED, KIND_HEAD = 1, 2, 3, 4, 5


def splitmix_next(state):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix64(a, b):
    return splitmix_next(a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & M64) + (a >> 2)) & M64))


def tensor_seed(base, kind, layer, expert):
    return mix64(base, ((kind << 48) ^ (layer << 16) ^ (expert + 1)) & M64)


def q4_roundtrip(w_bits):
    """bf16 weights as the engine streams them in Q4T mode: quantised on the
    GPU (kl_quantize_q4 = pyoracle.q4_quantize_tiled, bit-exact) and expanded
    back to bf16 by the fused-dequant GEMM (= q4_dequantize_tiled)."""
    rows, K = w_bits.shape
    return orc.bf16_bits(orc.q4_dequantize_tiled(orc.q4_quantize_tiled(w_bits), rows, K))


class TinyModel:
    def __init__(self, dims, weight_seed=7, q4_expert_layers=(), q4_attention_layers=()):
        self.D = D = dims
        self.seed = weight_seed
        d, f, E = D["d"], D["f"], D["E"]
        self.qkvw = (D["Hq"] + 2 * D["Hkv"]) * D["hd"]
        self.embed = orc.normal_bf16(D["V"] * d, tensor_seed(weight_seed, KIND_EMBED, 0, 0), 1.0).reshape(D["V"], d)
        self.head = orc.normal_bf16(D["V"] * d, tensor_seed(weight_seed, KIND_HEAD, 0, 0), 0.02).reshape(D["V"], d)
        self.norm = orc.bf16_bits(np.ones(d, np.float32))
        self.layers = []
        for l in range(D["L"]):
            a = orc.normal_bf16(self.qkvw * d + d * D["Hq"] * D["hd"], tensor_seed(weight_seed, KIND_ATTN, l, 0),
                                0.02)
            experts = []
            for e in range(E):
                w = orc.normal_bf16(3 * d * f, tensor_seed(weight_seed, KIND_EXPERT, l, e), 0.02)
                w13, w2 = w[: 2 * f * d].reshape(2 * f, d), w[2 * f * d:].reshape(d, f)
                if l in q4_expert_layers:
                    w13, w2 = q4_roundtrip(w13), q4_roundtrip(w2)
                experts.append((w13, w2))
            wqkv, wo = a[: self.qkvw * d].reshape(self.qkvw, d), a[self.qkvw * d:].reshape(d, D["Hq"] * D["hd"])
            if l in q4_attention_layers:
                wqkv, wo = q4_roundtrip(wqkv), q4_roundtrip(wo)
            fs = D.get("n_shared", 0) * D.get("f_shared", 0)
            g = orc.normal_bf16(E * d + 3 * d * fs, tensor_seed(weight_seed, KIND_GATE, l, 0), 0.02)
            shared = None
            if fs:  # router tensor = [router E x d | W13s (2 fs x d) | W2s (d x fs)] (engine gate slot)
                w13s = g[E * d: E * d + 2 * fs * d].reshape(2 * fs, d)
                w2s = g[E * d + 2 * fs * d:].reshape(d, fs)
                shared = (w13s, w2s)
            self.layers.append({
                "wqkv": wqkv,
                "wo": wo,
                "wg": np.ascontiguousarray(g[: E * d]).reshape(E, d),
                "experts": experts,
                "shared": shared,
            })

    def new_kv(self, n_seqs, cap):
        D = self.D
        size = n_seqs * cap * D["Hkv"] * D["hd"]
        return [(np.zeros(size, np.uint16), np.zeros(size, np.uint16)) for _ in range(D["L"])]

    def layer(self, l, h, step, n_batches, batch_size, prompt_len, kv, cap, sink, forced_idx=None):
        """One decoder layer on the whole batch group (rows batch-major,
        sequence-major). Returns (output hidden bf16 bits, routing ids)."""
        D, W = self.D, self.layers[l]
        hd, d = D["hd"], D["d"]
        tpb = batch_size * (prompt_len if step == 0 else 1)
        h = h.copy()
        kc, vc = kv[l]
        for b in range(n_batches):
            rows = slice(b * tpb, (b + 1) * tpb)
            hb = np.ascontiguousarray(h[rows])
            xa = orc.rmsnorm(hb, self.norm, D["eps"])
            qkv = orc.bf16_bits(orc.gemm_f32(xa, W["wqkv"]))
            if step == 0:
                pos = np.tile(np.arange(prompt_len, dtype=np.int32), batch_size)
                seq = np.repeat(np.arange(b * batch_size, (b + 1) * batch_size, dtype=np.int32), prompt_len)
                orc.rope_kv_append(qkv, D["Hq"], D["Hkv"], hd, pos, seq, D["theta"], kc, vc, cap, sink, prompt_len - 1)
                ao = orc.attn_prefill(qkv, batch_size, prompt_len, D["Hq"], D["Hkv"], hd, cap, sink, hd ** -0.5)
            else:
                pos = np.full(tpb, prompt_len + step - 1, np.int32)
                seq = np.arange(b * batch_size, (b + 1) * batch_size, dtype=np.int32)
                orc.rope_kv_append(qkv, D["Hq"], D["Hkv"], hd, pos, seq, D["theta"], kc, vc, cap, sink, -1)
                ao = orc.attn_decode(qkv, self.qkvw, pos, seq, D["Hq"], D["Hkv"], hd, kc, vc, cap, hd ** -0.5)
            h[rows] = orc.bf16_bits(orc.gemm_f32(ao, W["wo"]) + orc.bits_to_f32(hb))
        x2 = orc.rmsnorm(h, self.norm, D["eps"])
        logits, idx, w = orc.gate_topk(x2, W["wg"], D["k"], D.get("score_mode", 0))
        own_idx = idx.copy()
        if forced_idx is not None:
            idx = forced_idx.astype(np.int32).reshape(idx.shape)
            sel = np.take_along_axis(logits, idx, 1).astype(np.float32)
            if D.get("score_mode", 0) == 0:  # Mixtral: softmax over the k selected logits
                p = np.exp(sel - sel[:, :1])
                w = (p / p.sum(1, keepdims=True)).astype(np.float32)
            else:  # softmax over all E logits, weights of the selected ones (no renormalisation)
                mx = logits.max(1, keepdims=True).astype(np.float32)
                s = np.exp(logits.astype(np.float32) - mx).sum(1, keepdims=True)
                w = (np.exp(sel - mx) / s).astype(np.float32)
        if W["shared"] is not None:
            # h += shared SwiGLU FFN(x2): bf16 hidden, fp32 down projection + residual, one rounding.
            w13s, w2s = W["shared"]
            fs = w2s.shape[1]
            g = orc.gemm_f32(x2, np.ascontiguousarray(w13s[:fs])).astype(np.float64)
            u = orc.gemm_f32(x2, np.ascontiguousarray(w13s[fs:])).astype(np.float64)
            hs = orc.bf16_bits((g / (1.0 + np.exp(-g)) * u).astype(np.float32))
            h = orc.bf16_bits(orc.gemm_f32(hs, w2s) + orc.bits_to_f32(h))
        counts, offsets, pos_r, row_token = orc.permute(idx, D["E"])
        xp = np.ascontiguousarray(x2[row_token])
        y = np.empty_like(xp)
        for e in range(D["E"]):
            lo, hi = offsets[e], offsets[e + 1]
            if hi > lo:
                y[lo:hi] = orc.expert_ffn(np.ascontiguousarray(xp[lo:hi]), *W["experts"][e])
        return orc.combine(y, pos_r, w, h), own_idx, logits

    def greedy(self, h_last):
        x = orc.rmsnorm(h_last, self.norm, self.D["eps"])
        logits = orc.gemm_f32(x, self.head)
        return orc.bits_to_f32(orc.bf16_bits(logits)).argmax(1), logits
