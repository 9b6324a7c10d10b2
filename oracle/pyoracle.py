"""ctypes loader for oracle/liboracle.so (the CPU numeric oracle).

Test infrastructure only (see oracle/numerics.c header): imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs.
Arrays are numpy; bf16 values travel as uint16 bit patterns.
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_lib = C.CDLL(os.path.join(ROOT, "oracle", "liboracle.so"))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_P, _I, _L, _F = C.c_void_p, C.c_int, C.c_int64, C.c_float
_sigs = {
    "orc_gate_topk": [_P, _P, _I, _I, _I, _I, _I, _P, _P, _P],
    "orc_rmsnorm": [_P, _P, _L, _I, _F, _P],
    "orc_permute": [_P, _L, _I, _I, _P, _P, _P, _P],
    "orc_combine": [_P, _P, _P, _P, _L, _I, _I, _P],
    "orc_coact_update": [_P, _P, _L, _I, _I, _I, _P, _P],
    "orc_predict_scores": [_P, _P, _I, _I, _P],
    "orc_gemm_f32": [_P, _P, _L, _L, _L, _P],
    "orc_expert_ffn": [_P, _L, _I, _I, _P, _P, _P],
    "orc_rope_kv_append": [_P, _L, _I, _I, _I, _P, _P, _F, _P, _P, _I, _I, _I],
    "orc_attn_decode": [_P, _L, _P, _P, _L, _I, _I, _I, _P, _P, _I, _F, _P],
    "orc_attn_prefill": [_P, _I, _I, _I, _I, _I, _I, _I, _F, _P],
    "orc_fill_normal_bf16": [_P, _L, C.c_uint64, _F],
    "orc_f32_to_bf16": [_P, _L, _P],
    "orc_bf16_to_f32": [_P, _L, _P],
}
for name, args in _sigs.items():
    getattr(_lib, name).argtypes = args
    getattr(_lib, name).restype = None


def bf16_bits(x_f32):
    x = np.ascontiguousarray(x_f32, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    _lib.orc_f32_to_bf16(_p(x), x.size, _p(out))
    return out


def bits_to_f32(b):
    b = np.ascontiguousarray(b, dtype=np.uint16)
    out = np.empty(b.shape, dtype=np.float32)
    _lib.orc_bf16_to_f32(_p(b), b.size, _p(out))
    return out


def normal_bf16(n, seed, std):
    out = np.empty(n, dtype=np.uint16)
    _lib.orc_fill_normal_bf16(_p(out), n, seed, std)
    return out


def gate_topk(x2, wg, k, score_mode=0):
    T, d = x2.shape
    E = wg.shape[0]
    logits = np.empty((T, E), np.float32)
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float32)
    _lib.orc_gate_topk(_p(x2), _p(wg), T, d, E, k, score_mode, _p(logits), _p(idx), _p(w))
    return logits, idx, w


def rmsnorm(x, w, eps=1e-5):
    out = np.empty_like(x)
    _lib.orc_rmsnorm(_p(x), _p(w), x.shape[0], x.shape[1], eps, _p(out))
    return out


def permute(idx, E):
    T, k = idx.shape
    idx = np.ascontiguousarray(idx, np.int32)
    counts = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int32)
    pos = np.empty(T * k, np.int32)
    row_token = np.empty(T * k, np.int32)
    _lib.orc_permute(_p(idx), T, k, E, _p(counts), _p(offsets), _p(pos), _p(row_token))
    return counts, offsets, pos, row_token


def combine(y, pos, weight, resid):
    T, k = weight.shape
    out = np.empty_like(resid)
    _lib.orc_combine(_p(y), _p(pos), _p(weight), _p(resid), T, k, resid.shape[1], _p(out))
    return out


def coact_update(prev, cur, E, layer, table, marginal):
    T, k = cur.shape
    _lib.orc_coact_update(_p(prev), _p(cur), T, k, E, layer, _p(table), _p(marginal))


def predict_scores(hist, table, E, layer):
    score = np.empty(E, np.int64)
    _lib.orc_predict_scores(_p(hist), _p(table), E, layer, _p(score))
    return score


def gemm_f32(a, b):
    M, K = a.shape
    N = b.shape[0]
    c = np.empty((M, N), np.float32)
    _lib.orc_gemm_f32(_p(a), _p(b), M, N, K, _p(c))
    return c


def expert_ffn(x, w13, w2):
    M, d = x.shape
    f = w2.shape[1]
    y = np.empty((M, d), np.uint16)
    _lib.orc_expert_ffn(_p(x), M, d, f, _p(w13), _p(w2), _p(y))
    return y


def rope_kv_append(qkv, Hq, Hkv, hd, pos, seq, theta, kc, vc, cap, sink, chunk_last_pos=-1):
    _lib.orc_rope_kv_append(_p(qkv), qkv.shape[0], Hq, Hkv, hd, _p(pos), _p(seq), theta, _p(kc), _p(vc), cap, sink,
                            chunk_last_pos)


def attn_decode(q, q_stride, pos, seq, Hq, Hkv, hd, kc, vc, cap, scale):
    T = pos.shape[0]
    out = np.empty((T, Hq * hd), np.uint16)
    _lib.orc_attn_decode(_p(q), q_stride, _p(pos), _p(seq), T, Hq, Hkv, hd, _p(kc), _p(vc), cap, scale, _p(out))
    return out


def attn_prefill(qkv, n_seq, L, Hq, Hkv, hd, cap, sink, scale):
    out = np.empty((n_seq * L, Hq * hd), np.uint16)
    _lib.orc_attn_prefill(_p(qkv), n_seq, L, Hq, Hkv, hd, cap, sink, scale, _p(out))
    return out


# ---- 4-bit expert format (Q4T), restated from the reference quant.cpp ----
# fit_minmax (quant.cpp, QuantConfig{4, 64}): s = (hi - lo) / 15 in fp32,
# scale = fp16(s), zero = fp16(-lo / s); lo == hi -> (fp16(1), fp16(-lo)).
# code_of: clamp(round_half_away(double(w) / scale + zero), 0, 15).
# value_of: scale * (code - zero). Groups of 64 along K; Q4T stores the
# groups of each 128-row x 64-column tile as [128 x 32 B codes (element 2i in
# the low nibble of byte i) | 128 fp16 scales | 128 fp16 zeros].
Q4_CHUNK = 128 * 32 + 128 * 4


def q4_fit_minmax(groups_f32):
    """groups [n, 64] float32 -> (scale f16 [n], zero f16 [n])."""
    lo = groups_f32.min(axis=1)
    hi = groups_f32.max(axis=1)
    s = ((hi - lo).astype(np.float32) / np.float32(15.0)).astype(np.float32)
    same = lo == hi
    with np.errstate(divide="ignore", invalid="ignore"):
        z = (-lo / np.where(same, np.float32(1.0), s)).astype(np.float32)
    scale = np.where(same, np.float16(1.0), s.astype(np.float16))
    zero = np.where(same, (-lo).astype(np.float16), z.astype(np.float16))
    return scale.astype(np.float16), zero.astype(np.float16)


def q4_codes(groups_f32, scale, zero):
    x = groups_f32.astype(np.float64) / scale.astype(np.float64)[:, None] + zero.astype(np.float64)[:, None]
    q = np.floor(x + 0.5)  # std::round (half away from zero) for x >= -0.5; clamped below anyway
    return np.clip(q, 0, 15).astype(np.uint8)


def q4_quantize_tiled(w_bits):
    """bf16 bits [rows, K] -> Q4T bytes (min-max fit), the oracle of kl_quantize_q4."""
    rows, K = w_bits.shape
    KB = K // 64
    g = bits_to_f32(np.ascontiguousarray(w_bits)).reshape(rows, KB, 64)
    scale, zero = q4_fit_minmax(g.reshape(-1, 64))
    codes = q4_codes(g.reshape(-1, 64), scale, zero).reshape(rows, KB, 64)
    scale = scale.reshape(rows, KB)
    zero = zero.reshape(rows, KB)
    out = np.zeros(rows // 128 * KB * Q4_CHUNK, np.uint8)
    packed = (codes[:, :, 0::2] | (codes[:, :, 1::2] << 4)).astype(np.uint8)  # [rows, KB, 32]
    for rt in range(rows // 128):
        for kb in range(KB):
            base = (rt * KB + kb) * Q4_CHUNK
            blk = slice(rt * 128, rt * 128 + 128)
            out[base:base + 4096] = packed[blk, kb, :].reshape(-1)
            out[base + 4096:base + 4352] = np.ascontiguousarray(scale[blk, kb]).view(np.uint8)
            out[base + 4352:base + 4608] = np.ascontiguousarray(zero[blk, kb]).view(np.uint8)
    return out


def q4_dequantize_tiled(q, rows, K):
    """Q4T -> float32 [rows, K] (value_of in fp32: one rounding of the exact product)."""
    KB = K // 64
    out = np.empty((rows, K), np.float32)
    for rt in range(rows // 128):
        for kb in range(KB):
            base = (rt * KB + kb) * Q4_CHUNK
            codes = q[base:base + 4096].reshape(128, 32)
            c = np.empty((128, 64), np.float32)
            c[:, 0::2] = codes & 15
            c[:, 1::2] = codes >> 4
            sc = np.ascontiguousarray(q[base + 4096:base + 4352]).view(np.float16).astype(np.float32)
            zr = np.ascontiguousarray(q[base + 4352:base + 4608]).view(np.float16).astype(np.float32)
            out[rt * 128:rt * 128 + 128, kb * 64:kb * 64 + 64] = (sc[:, None] * (c - zr[:, None])).astype(np.float32)
    return out
