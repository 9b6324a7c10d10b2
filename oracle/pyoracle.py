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
