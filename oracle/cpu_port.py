"""CPU port of the decode step, built from the C numeric oracle — the CPU
baseline of bench.py (cpu_baseline, kind "port") and its --impl reference arm.

The reference (proj/) has no numeric CPU path: its only "execution" is the
discrete-event simulator (simulator.cpp:70-287), which prices ops instead of
computing them. The CPU counterpart of the B200 decode step is therefore this
restatement: per layer, n attention blocks (RMSNorm, QKV, RoPE, GQA decode
attention over the retained KV, O projection + residual), the router (RMSNorm,
gate, top-k), the expert-major permutation, every active expert's SwiGLU FFN
and the weighted combine — exactly the B200 kernels' arithmetic in fp32/bf16
on host cores with OpenMP (all threads the box gives us).

Bounded samples: `measure` times one full layer of one decode step at the
workload's shape (n batches x batch_size tokens) and extrapolates to all
layers (bench.py's cpu_baseline); `StepSample` runs WHOLE decode steps of one
batch through every layer (bench.py --impl reference), the layers aliased onto
one layer's weights and KV (a layer's 2.8 GB of weights exceeds every CPU
cache, so each layer streams them from DRAM either way).
Weights/KV are synthetic bf16 from the same SplitMix64 stream family.
"""
import os
import time

import numpy as np

from oracle import pyoracle as orc


def mixtral_dims(preset):
    return {
        "mixtral-8x7b": dict(L=32, d=4096, f=14336, Hq=32, Hkv=8, hd=128, E=8, k=2),
        "mixtral-8x22b": dict(L=56, d=6144, f=16384, Hq=48, Hkv=8, hd=128, E=8, k=2),
        "tiny": dict(L=4, d=512, f=1792, Hq=8, Hkv=2, hd=64, E=8, k=2),
    }[preset]


class LayerSample:
    """One decoder layer's weights + KV for `seqs` sequences (synthetic)."""

    def __init__(self, dims, n_batches, batch_size, cap, seed=7):
        D = dims
        self.D, self.n, self.bs, self.cap = D, n_batches, batch_size, cap
        qkvw = (D["Hq"] + 2 * D["Hkv"]) * D["hd"]
        d, f = D["d"], D["f"]
        self.wqkv = orc.normal_bf16(qkvw * d, seed + 1, 0.02).reshape(qkvw, d)
        self.wo = orc.normal_bf16(d * D["Hq"] * D["hd"], seed + 2, 0.02).reshape(d, D["Hq"] * D["hd"])
        self.wg = orc.normal_bf16(D["E"] * d, seed + 3, 0.02).reshape(D["E"], d)
        self.norm = orc.bf16_bits(np.ones(d, np.float32))
        self.w13 = [orc.normal_bf16(2 * f * d, seed + 10 + e, 0.02).reshape(2 * f, d) for e in range(D["E"])]
        self.w2 = [orc.normal_bf16(d * f, seed + 40 + e, 0.02).reshape(d, f) for e in range(D["E"])]
        seqs = n_batches * batch_size
        self.kc = orc.normal_bf16(seqs * cap * D["Hkv"] * D["hd"], seed + 5, 1.0)
        self.vc = orc.normal_bf16(seqs * cap * D["Hkv"] * D["hd"], seed + 6, 1.0)
        self.h = orc.normal_bf16(seqs * d, seed + 8, 1.0).reshape(seqs, d)

    def decode_layer(self, pos_value, sink=4):
        """One decode step through this layer for all n*bs sequences (in place)."""
        D, n, bs = self.D, self.n, self.bs
        d, hd = D["d"], D["hd"]
        qkvw = (D["Hq"] + 2 * D["Hkv"]) * hd
        scale = hd ** -0.5
        for b in range(n):
            rows = slice(b * bs, (b + 1) * bs)
            hb = np.ascontiguousarray(self.h[rows])
            xa = orc.rmsnorm(hb, self.norm)
            qkv = orc.bf16_bits(orc.gemm_f32(xa, self.wqkv))
            pos = np.full(bs, pos_value, np.int32)
            seq = np.arange(b * bs, (b + 1) * bs, dtype=np.int32)
            orc.rope_kv_append(qkv, D["Hq"], D["Hkv"], hd, pos, seq, 1e6, self.kc, self.vc, self.cap, sink)
            ao = orc.attn_decode(qkv, qkvw, pos, seq, D["Hq"], D["Hkv"], hd, self.kc, self.vc, self.cap, scale)
            o = orc.gemm_f32(ao, self.wo) + orc.bits_to_f32(hb)
            self.h[rows] = orc.bf16_bits(o)
        x2 = orc.rmsnorm(self.h, self.norm)
        _, idx, w = orc.gate_topk(x2, self.wg, D["k"])
        counts, offsets, pos_r, row_token = orc.permute(idx, D["E"])
        xp = np.ascontiguousarray(x2[row_token])
        y = np.empty_like(xp)
        for e in range(D["E"]):
            lo, hi = offsets[e], offsets[e + 1]
            if hi > lo:
                y[lo:hi] = orc.expert_ffn(np.ascontiguousarray(xp[lo:hi]), self.w13[e], self.w2[e])
        self.h = orc.combine(y, pos_r, w, self.h)


class StepSample:
    """Whole decode steps: one batch of `batch_size` sequences through all L
    layers (the layers share one LayerSample's weights and KV)."""

    def __init__(self, preset="mixtral-8x7b", batch_size=64, cap=260):
        self.D = mixtral_dims(preset)
        self.layer = LayerSample(self.D, 1, batch_size, cap)
        self.tokens = batch_size

    def decode_step(self, pos_value=600):
        for _ in range(self.D["L"]):
            self.layer.decode_layer(pos_value)


def measure(preset="mixtral-8x7b", n_batches=8, batch_size=64, cap=260, repeats=1, warmup=0):
    """Seconds per full decode step (extrapolated from one timed layer)."""
    D = mixtral_dims(preset)
    t_setup = time.perf_counter()
    layer = LayerSample(D, n_batches, batch_size, cap)
    setup = time.perf_counter() - t_setup
    for _ in range(warmup):
        layer.decode_layer(600)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        layer.decode_layer(600)
        times.append(time.perf_counter() - t0)
    per_layer = float(np.median(times))
    return {
        "layer_seconds": per_layer,
        "step_seconds": per_layer * D["L"],
        "tokens_per_step": n_batches * batch_size,
        "tok_s": n_batches * batch_size / (per_layer * D["L"]),
        "setup_seconds": setup,
        "cores": os.cpu_count(),
        "sample": f"1 of {D['L']} layers of one {preset} decode step ({n_batches}x{batch_size} tokens, "
                  f"{cap} retained KV slots), extrapolated x{D['L']}",
    }
