"""ctypes bindings for include/klotski/kernels.h (the kernel C-ABI).

Every function takes torch CUDA tensors, passes raw pointers + sizes to the
C entry point on the current torch stream (or an explicit `stream` handle)
and raises KernelError on a non-zero return code. No CPU fallback exists.
"""
import ctypes as C

import torch

from . import load_native

_lib = load_native()

_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_F = C.c_float
KL_EUNSUPPORTED = -2  # klotski/kernels.h
_U64 = C.c_uint64


def _sig(name, args, res=C.c_int):
    fn = getattr(_lib, name)
    fn.argtypes = args
    fn.restype = res
    return fn


_lib.kl_error_string.restype = C.c_char_p
_lib.kl_error_string.argtypes = [_I]
_gemm = _sig("kl_gemm_bf16", [_P, _L, _L, _I, _I, _P, _I, _P, _I, _P, _I, _P, _L, _P])
_gemm_ws = _sig("kl_gemm_workspace_bytes", [_I, _I, _I, _I], C.c_int64)
_ffn = _sig("kl_expert_ffn", [_P, _L, _L, _I, _I, _I, _P, _P, _P, _P, _P, _L, _P])
_ffn_kb = _sig("kl_expert_ffn_kb", [_P, _L, _L, _I, _I, _I, _P, _P, _P, _P, _P, _L, _P])
_gemm_kb = _sig("kl_gemm_bf16_kb", [_P, _L, _L, _I, _I, _P, _I, _P, _I, _P, _I, _P, _L, _P])
_kblock = _sig("kl_weights_kblock", [_P, _L, _L, _P, _P])
_gate = _sig("kl_gate_topk", [_P, _P, _P, _I, _I, _I, _I, _F, _I, _P, _P, _P, _P, _P, _P, _P])
_perm_ws = _sig("kl_permute_workspace_bytes", [_L, _I], C.c_int64)
_perm = _sig("kl_permute", [_P, _L, _I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _P])
_comb = _sig("kl_combine", [_P, _P, _P, _P, _L, _I, _I, _P, _P])
_comb_def = _sig("kl_combine_deferred", [_P, _I, _L, _P, _P, _P, _L, _I, _I, _P, _P])
_ffn_def = _sig("kl_expert_ffn_kb_deferred", [_P, _L, _L, _I, _I, _I, _P, _P, _P, _P, _L, _I, _P, _L, _P])
_ffn_def_splits = _sig("kl_expert_ffn_deferred_splits", [_I, _I, _I])
_gemm_def_splits = _sig("kl_gemm_deferred_splits", [_I, _I, _I])
_gemm_def = _sig("kl_gemm_bf16_deferred", [_P, _L, _L, _I, _I, _P, _I, _I, _P, _L, _I, _P, _L, _P])
_gate_def = _sig("kl_gate_topk_deferred", [_P, _P, _I, _L, _P, _P, _I, _I, _I, _I, _F, _I, _P, _P, _P, _P, _P, _P,
                                           _P])
_rope_def = _sig("kl_rope_kv_append_deferred", [_P, _I, _L, _P, _L, _I, _I, _I, _P, _P, _F, _P, _P, _I, _I, _I, _P])
_coact = _sig("kl_coact_update", [_P, _P, _L, _I, _I, _I, _P, _P, _P])
_pred = _sig("kl_predict_scores", [_P, _P, _I, _I, _P, _P])
_rms = _sig("kl_rmsnorm", [_P, _P, _L, _I, _F, _P, _P])
_rope = _sig("kl_rope_kv_append", [_P, _L, _I, _I, _I, _P, _P, _F, _P, _P, _I, _I, _I, _P])
_rms_tab = _sig("kl_rmsnorm_rope_table", [_P, _P, _L, _I, _F, _P, _P, _F, _I, _P, _P])
_qkv_rope = _sig("kl_gemm_bf16_qkv_rope", [_P, _L, _L, _I, _I, _P, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _I, _I, _I,
                                           _P, _L, _P])
_dec = _sig("kl_attn_decode", [_P, _L, _P, _P, _L, _I, _I, _I, _P, _P, _I, _I, _F, _P, _P])
_dec_ws_bytes = _sig("kl_attn_decode_workspace_bytes", [_L, _I, _I, _I], C.c_int64)
_dec_ws = _sig("kl_attn_decode_ws", [_P, _L, _P, _P, _L, _I, _I, _I, _P, _P, _I, _I, _F, _P, _P, _L, _P])
_dec_ws2 = _sig("kl_attn_decode_ws2", [_P, _L, _P, _P, _L, _I, _I, _I, _P, _P, _L, _I, _I, _F, _P, _P, _L, _P])
_pre = _sig("kl_attn_prefill", [_P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _P])
_fill = _sig("kl_fill_normal_bf16", [_P, _L, _U64, _F, _P])
_tune = _sig("kl_tune", [_I, _I])
_q4_bytes = _sig("kl_q4_bytes", [_L, _L], C.c_int64)
_q4_quant = _sig("kl_quantize_q4", [_P, _L, _L, _P, _P])
_q4_dequant = _sig("kl_dequantize_q4", [_P, _L, _L, _P, _P])
_q4_ws = _sig("kl_gemm_q4_workspace_bytes", [_I, _I, _I, _I], C.c_int64)
_q4_gemm = _sig("kl_gemm_q4", [_P, _L, _L, _I, _I, _P, _I, _P, _I, _P, _I, _P, _L, _P])
_q4_ffn = _sig("kl_expert_ffn_q4", [_P, _L, _L, _I, _I, _I, _P, _P, _P, _P, _P, _L, _P])
abi_version = _sig("kl_abi_version", [])

TUNE_STREAM_GEMM = 0  # weight-streaming decode GEMM path on/off
TUNE_STREAM_NMMA = 1  # 128-row weight sub-tiles per activation tile (1 or 2)
TUNE_STREAM_STAGES = 2
TUNE_STREAM_HINT = 3
TUNE_STREAM_CTAS_PER_SM = 4
TUNE_PDL = 5
TUNE_PREFILL_TC = 6
TUNE_STREAM_WHOLE_TILES = 7
TUNE_GEMM_PERSISTENT = 8
TUNE_ROPE_TOKEN_BLOCKS = 11  # RoPE/KV append: block per token (1) or thread per element (0)
TUNE_STREAM_KBLOCKS_PER_STAGE = 12  # weight-streaming GEMM k-blocks per stage: 1, 2 (if >= 3 stages), 3 (default: 2 if >= 2 stages)
TUNE_STREAM_EVEN_SPLIT = 13  # weight-streaming GEMM: equal (1) or near-equal (2) k-splits per tile
TUNE_STREAM_FUSED_FIXUP = 16  # weight-streaming GEMM: owners add split partials in the epilogue pass
TUNE_DECODE_STAGES = 21  # tensor-core decode attention: ring stages (0 = default)
TUNE_ATTN_KV_EVICT_FIRST = 19  # decode attention: K/V loads L2 evict-first
TUNE_DECODE_HG = 18  # tensor-core decode attention: KV heads per work item (0 = auto)
TUNE_DECODE_MMA = 9  # persistent mma.sync split-KV decode attention (1) or per-chunk CUDA-core kernel (0)


def tune(knob, value):
    """Process-wide kernel tuning knob (kl_tune); for tests and benchmarks."""
    _chk(_tune(knob, value), "kl_tune")
device_supported = _sig("kl_device_supported", [])


class KernelError(RuntimeError):
    pass


def _chk(rc, name):
    if rc != 0:
        raise KernelError(f"{name}: {_lib.kl_error_string(rc).decode()} (code {rc})")


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _s(stream):
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    return C.c_void_p(stream)


_ws_cache = {}


def workspace(nbytes, device):
    """Reusable fp32 split-K workspace (caller-owned per the C-ABI)."""
    key = (str(device),)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def workspace_bytes(M, N, K, epilogue=0):
    return int(_gemm_ws(M, N, K, epilogue))


def weights_kblock(w, stream=None):
    """Row-major bf16 [rows, cols] -> the K-blocked layout (kl_weights_kblock);
    returned with the same shape (the bytes are reordered, not the meaning)."""
    rows, cols = w.shape
    out = torch.empty_like(w)
    _chk(_kblock(_p(w), rows, cols, _p(out), _s(stream)), "kl_weights_kblock")
    return out


def gemm(a, b, c=None, residual=None, epilogue=0, row_offset=0, m=None, stream=None, split_k=True, ws_bytes=None,
         kblocked=False):
    """C = A[row_offset:row_offset+m] @ B^T (bf16, fp32 accumulate) on tcgen05.
    kblocked: b holds the K-blocked layout of the [N, K] weights."""
    m = a.shape[0] - row_offset if m is None else m
    K = a.shape[1]
    N = b.shape[0]
    n_out = N // 2 if epilogue == 2 else N
    if c is None:
        c = torch.empty(m, n_out, dtype=torch.bfloat16, device=a.device)
    wsb = workspace_bytes(m, N, K, epilogue) if split_k else 0
    if ws_bytes is not None and split_k:
        wsb = int(ws_bytes)
    ws = workspace(wsb, a.device) if wsb else None
    fn = _gemm_kb if kblocked else _gemm
    _chk(fn(_p(a), a.shape[0], row_offset, m, K, _p(b), N, _p(c), c.stride(0), _p(residual), epilogue, _p(ws),
            wsb, _s(stream)), "kl_gemm_bf16_kb" if kblocked else "kl_gemm_bf16")
    return c


def expert_ffn(xp, row_offset, m, w13, w2, y, h_scratch, stream=None, split_k=True, kblocked=False):
    """One expert's SwiGLU FFN (kl_expert_ffn); kblocked: w13 [2f, d] and
    w2 [d, f] hold the K-blocked layout (kl_expert_ffn_kb)."""
    d = xp.shape[1]
    f = w2.shape[1]
    wsb = max(workspace_bytes(m, 2 * f, d, 2), workspace_bytes(m, d, f, 0)) if split_k else 0
    ws = workspace(wsb, xp.device) if wsb else None
    fn = _ffn_kb if kblocked else _ffn
    _chk(fn(_p(xp), xp.shape[0], row_offset, m, d, f, _p(w13), _p(w2), _p(h_scratch), _p(y), _p(ws), wsb,
            _s(stream)), "kl_expert_ffn_kb" if kblocked else "kl_expert_ffn")


def q4_bytes(rows, K):
    return int(_q4_bytes(rows, K))


def quantize_q4(w, stream=None):
    """bf16 [rows, K] -> Q4T bytes (uint8 tensor), min-max fit per group of 64."""
    rows, K = w.shape
    out = torch.empty(q4_bytes(rows, K), dtype=torch.uint8, device=w.device)
    _chk(_q4_quant(_p(w), rows, K, _p(out), _s(stream)), "kl_quantize_q4")
    return out


def dequantize_q4(q, rows, K, stream=None):
    out = torch.empty(rows, K, dtype=torch.bfloat16, device=q.device)
    _chk(_q4_dequant(_p(q), rows, K, _p(out), _s(stream)), "kl_dequantize_q4")
    return out


def gemm_q4(a, bq, N, c=None, residual=None, epilogue=0, row_offset=0, m=None, stream=None):
    """C = A[row_offset:row_offset+m] @ dequant(Bq)^T with the dequant fused into the GEMM producer."""
    m = a.shape[0] - row_offset if m is None else m
    K = a.shape[1]
    n_out = N // 2 if epilogue == 2 else N
    if c is None:
        c = torch.empty(m, n_out, dtype=torch.bfloat16, device=a.device)
    wsb = int(_q4_ws(m, N, K, epilogue))
    ws = workspace(wsb, a.device)
    _chk(_q4_gemm(_p(a), a.shape[0], row_offset, m, K, _p(bq), N, _p(c), c.stride(0), _p(residual), epilogue, _p(ws),
                  wsb, _s(stream)), "kl_gemm_q4")
    return c


def expert_ffn_q4(xp, row_offset, m, w13q, w2q, d, f, y, h_scratch, stream=None):
    wsb = max(int(_q4_ws(m, 2 * f, d, 2)), int(_q4_ws(m, d, f, 0)))
    ws = workspace(wsb, xp.device)
    _chk(_q4_ffn(_p(xp), xp.shape[0], row_offset, m, d, f, _p(w13q), _p(w2q), _p(h_scratch), _p(y), _p(ws), wsb,
                 _s(stream)), "kl_expert_ffn_q4")


def gate_topk(h, norm_w, wg, k, eps=1e-5, score_mode=0, x2=None, logits=None, hist=None, first_pos=None,
              stream=None):
    T, d = h.shape
    E = wg.shape[0]
    dev = h.device
    x2 = torch.empty_like(h) if x2 is None else x2
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    _chk(_gate(_p(h), _p(norm_w), _p(wg), T, d, E, k, eps, score_mode, _p(x2), _p(logits), _p(idx), _p(w),
               _p(hist), _p(first_pos), _s(stream)), "kl_gate_topk")
    return x2, idx, w


def permute(idx, E, x2=None, stream=None, with_rows=True):
    T, k = idx.shape
    dev = idx.device
    R = T * k
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    offsets = torch.empty(E + 1, dtype=torch.int32, device=dev)
    pos = torch.empty(R, dtype=torch.int32, device=dev)
    row_token = torch.empty(R, dtype=torch.int32, device=dev)
    ws = torch.empty(int(_perm_ws(R, E)), dtype=torch.uint8, device=dev)
    xp = None
    d = 0
    if x2 is not None and with_rows:
        d = x2.shape[1]
        xp = torch.empty(R, d, dtype=x2.dtype, device=dev)
    _chk(_perm(_p(idx), T, k, E, _p(x2), d, _p(counts), _p(offsets), _p(pos), _p(row_token), _p(xp), _p(ws),
               _s(stream)), "kl_permute")
    return counts, offsets, pos, row_token, xp


def combine(y, pos, weight, resid, out=None, stream=None):
    T, k = weight.shape
    d = resid.shape[1]
    out = torch.empty_like(resid) if out is None else out
    _chk(_comb(_p(y), _p(pos), _p(weight), _p(resid), T, k, d, _p(out), _s(stream)), "kl_combine")
    return out


def expert_ffn_deferred_splits(M, d, f):
    return int(_ffn_def_splits(M, d, f))


def expert_ffn_deferred(xp, row_offset, m, w13, w2, y_part, h_scratch, splits, stream=None):
    """kl_expert_ffn_kb_deferred: K-blocked weights, down-projection splits
    left as fp32 partials in y_part [splits, rows, d]."""
    d = xp.shape[1]
    f = w2.shape[1]
    wsb = workspace_bytes(m, 2 * f, d, 2)
    ws = workspace(max(wsb, 1024), xp.device)
    _chk(_ffn_def(_p(xp), xp.shape[0], row_offset, m, d, f, _p(w13), _p(w2), _p(h_scratch), _p(y_part),
                  y_part.shape[1], splits, _p(ws), max(wsb, 1024), _s(stream)), "kl_expert_ffn_kb_deferred")


def gemm_deferred_splits(M, N, K):
    return int(_gemm_def_splits(M, N, K))


def gemm_deferred(a, b, c_part, splits, row_offset=0, m=None, kblocked=False, stream=None):
    """kl_gemm_bf16_deferred: fp32 split partials into c_part [splits, rows, N]."""
    m = a.shape[0] - row_offset if m is None else m
    N, K = b.shape[0], a.shape[1]
    _chk(_gemm_def(_p(a), a.shape[0], row_offset, m, K, _p(b), N, int(kblocked), _p(c_part), c_part.shape[1], splits,
                   None, 0, _s(stream)), "kl_gemm_bf16_deferred")
    return c_part


def gate_topk_deferred(h, h_part, splits, norm_w, wg, k, eps=1e-5, score_mode=0, x2=None, logits=None, hist=None,
                       first_pos=None, stream=None):
    """kl_gate_topk_deferred: completes h in place from o-proj split partials
    h_part [splits, rows, d], then the router; returns (x2, idx, weight)."""
    T, d = h.shape
    E = wg.shape[0]
    x2 = torch.empty_like(h) if x2 is None else x2
    idx = torch.empty(T, k, dtype=torch.int32, device=h.device)
    wt = torch.empty(T, k, dtype=torch.float32, device=h.device)
    _chk(_gate_def(_p(h), _p(h_part), splits, h_part.shape[1], _p(norm_w), _p(wg), T, d, E, k, eps, score_mode, _p(x2),
                   _p(logits), _p(idx), _p(wt), _p(hist), _p(first_pos), _s(stream)), "kl_gate_topk_deferred")
    return x2, idx, wt


def rope_kv_append_deferred(qkv_part, splits, qkv, Hq, Hkv, hd, pos, seq, theta, k_cache, v_cache, cap, sink,
                            chunk_last_pos=-1, stream=None):
    _chk(_rope_def(_p(qkv_part), splits, qkv_part.shape[1], _p(qkv), qkv.shape[0], Hq, Hkv, hd, _p(pos), _p(seq),
                   theta, _p(k_cache), _p(v_cache), cap, sink, chunk_last_pos, _s(stream)),
         "kl_rope_kv_append_deferred")


def combine_deferred(y_part, splits, pos, weight, resid, out=None, stream=None):
    T, k = weight.shape
    d = resid.shape[1]
    out = torch.empty_like(resid) if out is None else out
    _chk(_comb_def(_p(y_part), splits, y_part.shape[1], _p(pos), _p(weight), _p(resid), T, k, d, _p(out), _s(stream)),
         "kl_combine_deferred")
    return out


def coact_update(prev, cur, E, layer, table, marginal, stream=None):
    T, k = cur.shape
    _chk(_coact(_p(prev), _p(cur), T, k, E, layer, _p(table), _p(marginal), _s(stream)), "kl_coact_update")


def predict_scores(hist, table, E, layer, stream=None):
    score = torch.empty(E, dtype=torch.int64, device=hist.device)
    _chk(_pred(_p(hist), _p(table), E, layer, _p(score), _s(stream)), "kl_predict_scores")
    return score


def rmsnorm(x, w, eps=1e-5, out=None, stream=None):
    out = torch.empty_like(x) if out is None else out
    _chk(_rms(_p(x), _p(w), x.shape[0], x.shape[1], eps, _p(out), _s(stream)), "kl_rmsnorm")
    return out


def rope_kv_append(qkv, Hq, Hkv, hd, pos, seq, theta, k_cache, v_cache, cap, sink, chunk_last_pos=-1,
                   stream=None):
    _chk(_rope(_p(qkv), qkv.shape[0], Hq, Hkv, hd, _p(pos), _p(seq), theta, _p(k_cache), _p(v_cache), cap, sink,
               chunk_last_pos, _s(stream)), "kl_rope_kv_append")


def rmsnorm_rope_table(x, w, pos, theta, hd, eps=1e-5, out=None, table=None, stream=None):
    """kl_rmsnorm_rope_table: RMSNorm of decode-sized x plus each row's RoPE
    (cos, sin) table [T, hd/2, 2] fp32 for qkv_rope."""
    out = torch.empty_like(x) if out is None else out
    if table is None:
        table = torch.empty(x.shape[0], hd // 2, 2, dtype=torch.float32, device=x.device)
    _chk(_rms_tab(_p(x), _p(w), x.shape[0], x.shape[1], eps, _p(out), _p(pos), theta, hd, _p(table), _s(stream)),
         "kl_rmsnorm_rope_table")
    return out, table


def qkv_rope(a, b, Hq, Hkv, hd, table, pos, seq, k_cache, v_cache, cap, sink, chunk_last_pos=-1, c=None,
             row_offset=0, m=None, stream=None):
    """kl_gemm_bf16_qkv_rope: the QKV GEMM with RoPE + KV append in its
    epilogue. Returns c, or None when the shape is not on the fused path
    (KL_EUNSUPPORTED: the caller runs gemm + rope_kv_append)."""
    m = a.shape[0] - row_offset if m is None else m
    N = b.shape[0]
    c = torch.empty(m, N, dtype=torch.bfloat16, device=a.device) if c is None else c
    wsb = workspace_bytes(m, N, a.shape[1], 0)
    ws = workspace(max(wsb, 1024), a.device)
    rc = _qkv_rope(_p(a), a.shape[0], row_offset, m, a.shape[1], _p(b), Hq, Hkv, hd, _p(c), c.stride(0), _p(table),
                   _p(pos), _p(seq), _p(k_cache), _p(v_cache), cap, sink, chunk_last_pos, _p(ws), max(wsb, 1024),
                   _s(stream))
    if rc == KL_EUNSUPPORTED:
        return None
    _chk(rc, "kl_gemm_bf16_qkv_rope")
    return c


def attn_decode(q, q_stride, pos, seq, Hq, Hkv, hd, k_cache, v_cache, cap, sink, scale, out, stream=None):
    T = pos.shape[0]
    _chk(_dec(_p(q), q_stride, _p(pos), _p(seq), T, Hq, Hkv, hd, _p(k_cache), _p(v_cache), cap, sink, scale,
              _p(out), _s(stream)), "kl_attn_decode")
    return out


def attn_decode_split(q, q_stride, pos, seq, Hq, Hkv, hd, k_cache, v_cache, cap, sink, scale, out, stream=None):
    """Split-KV decode attention (kl_attn_decode_ws) with a cached workspace."""
    T = pos.shape[0]
    wsb = int(_dec_ws_bytes(T, Hq, hd, cap))
    ws = workspace(wsb, q.device)
    cache_seqs = k_cache.numel() // (cap * Hkv * hd)  # the cache's extent: the tensor-core kernel's TMA bounds
    _chk(_dec_ws2(_p(q), q_stride, _p(pos), _p(seq), T, Hq, Hkv, hd, _p(k_cache), _p(v_cache), cache_seqs, cap, sink,
                  scale, _p(out), _p(ws), wsb, _s(stream)), "kl_attn_decode_ws2")
    return out


def attn_prefill(qkv, n_seq, L, Hq, Hkv, hd, cap, sink, scale, out, stream=None):
    _chk(_pre(_p(qkv), n_seq, L, Hq, Hkv, hd, cap, sink, scale, _p(out), _s(stream)), "kl_attn_prefill")
    return out


def fill_normal(t, seed, std, stream=None):
    _chk(_fill(_p(t), t.numel(), seed, std, _s(stream)), "kl_fill_normal_bf16")
    return t
