"""Decode-shaped microbenchmarks of every kernel on the Mixtral-8x7B path
(through the C-ABI), timed with CUDA events on the launching stream after
warm-up, inputs larger than L2 where it matters (each expert call uses a
different 352 MB weight buffer). Also the target for `ncu --set full`.

    python tools/profile_kernels.py [--only ffn] [--iters N] [--json out.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402

d, f, E, k, Hq, Hkv, hd = 4096, 14336, 8, 2, 32, 8, 128
bs, n = 64, 8
T = bs * n


TRACE = False


def dump_trace(label):
    """Per-CTA phase timestamps of the last weight-streaming GEMM launch."""
    if not TRACE:
        return
    import ctypes
    import numpy as np
    buf = (ctypes.c_ulonglong * (256 * 12))()
    K._lib.kl_stream_trace(buf, 256)
    a = np.array(buf, dtype=np.float64).reshape(256, 12)[:148]
    t0 = a[:, 0][a[:, 0] > 0].min()
    rel = (a - t0) / 1e3
    rel[a == 0] = np.nan
    names = ["start", "mma0", "mma_end", "epi_last", "flags_ok", "landed", "sums_done", "end", "contrib0",
             "published", "staged", "stored"]
    print(f"trace {label} (us from first CTA start)")
    for i, nm in enumerate(names):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {nm:10s} med {np.nanmedian(col):7.2f}  min {np.nanmin(col):7.2f}  max {np.nanmax(col):7.2f}")


GAP_MS = 0.0


def timed(fn, iters, stream):
    if GAP_MS > 0:
        # Idle gaps between launches (as inside the link-bound decode step):
        # per-launch event times, median.
        # The stream is gated by a spin kernel on a host flag, so the timed
        # launch is already queued when the GPU wakes up (no host latency).
        import ctypes
        import time
        flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        for _ in range(3):
            fn(0)
        ts = []
        for i in range(iters):
            torch.cuda.synchronize()
            flag[0] = 0
            K._lib.kl_debug_spin_flag(ctypes.c_void_p(flag.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(i)
            b.record(stream)
            time.sleep(GAP_MS / 1e3)
            flag[0] = 1
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        return ts[len(ts) // 2] * 1e-3
    if TRACE:
        import ctypes
        buf = (ctypes.c_ulonglong * (256 * 12))()
        K._lib.kl_stream_trace(buf, 256)  # read + clear
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    if TRACE:
        import ctypes
        buf = (ctypes.c_ulonglong * (256 * 12))()
        K._lib.kl_stream_trace(buf, 256)  # clear: the trace shows the last timed launch only
    s.record(stream)
    for i in range(iters):
        fn(i)
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def timed_graph(fn, iters):
    """Device time per call with host overhead removed: `iters` calls
    captured once into a CUDA graph, replayed 3 times."""
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (3 * iters) * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rows", type=int, default=128)
    ap.add_argument("--json", default="")
    ap.add_argument("--nmma", type=int, default=1, help="weight sub-tiles per activation tile (stream GEMM)")
    ap.add_argument("--no-stream", action="store_true", help="disable the weight-streaming decode GEMM path")
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--hint", type=int, default=1)
    ap.add_argument("--ctas", type=int, default=1)
    ap.add_argument("--debug", type=int, default=0)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--persist", type=int, default=1)
    ap.add_argument("--ks", type=int, default=3, help="stream GEMM k-blocks per stage (knob 1|2|3)")
    ap.add_argument("--even", type=int, default=2, help="stream GEMM tile-aligned k-splits: 1 equal only, 2 near-equal too")
    ap.add_argument("--whole", type=int, default=70, help="whole-tile grid when tiles >= pct%% of SMs")
    ap.add_argument("--gap-ms", type=float, default=0.0, help="host sleep between timed launches")
    ap.add_argument("--split", type=int, default=-1, help="stream GEMM even-split mode (-1 = default)")
    ap.add_argument("--fused-fixup", type=int, default=-1, help="stream GEMM owners add partials in the epilogue pass")
    ap.add_argument("--kv-evict-first", type=int, default=-1, help="decode attention K/V loads evict-first")
    ap.add_argument("--decode-stages", type=int, default=-1, help="decode attention ring stages (0 = default)")
    ap.add_argument("--decode-hg", type=int, default=-1, help="decode attention KV heads per work item (0 = auto)")
    ap.add_argument("--kb", type=int, default=1, help="expert weights in the K-blocked layout (the engine's)")
    ap.add_argument("--h2d", action="store_true", help="keep a pinned-host -> HBM copy running on a side stream")
    args = ap.parse_args()
    K.tune(99, args.debug)
    K.tune(K.TUNE_PDL, args.pdl)
    K.tune(K.TUNE_STREAM_WHOLE_TILES, args.whole)
    K.tune(K.TUNE_GEMM_PERSISTENT, args.persist)
    K.tune(K.TUNE_STREAM_KBLOCKS_PER_STAGE, args.ks)
    K.tune(K.TUNE_STREAM_EVEN_SPLIT, args.even if args.split < 0 else args.split)
    if args.fused_fixup >= 0:
        K.tune(K.TUNE_STREAM_FUSED_FIXUP, args.fused_fixup)
    if args.kv_evict_first >= 0:
        K.tune(K.TUNE_ATTN_KV_EVICT_FIRST, args.kv_evict_first)
    if args.decode_stages >= 0:
        K.tune(K.TUNE_DECODE_STAGES, args.decode_stages)
    if args.decode_hg >= 0:
        K.tune(K.TUNE_DECODE_HG, args.decode_hg)
    global TRACE, GAP_MS
    GAP_MS = args.gap_ms
    TRACE = bool(args.debug & 128)
    K.tune(K.TUNE_STREAM_STAGES, args.stages)
    K.tune(K.TUNE_STREAM_HINT, args.hint)
    K.tune(K.TUNE_STREAM_CTAS_PER_SM, args.ctas)
    K.tune(K.TUNE_STREAM_NMMA, args.nmma)
    K.tune(K.TUNE_STREAM_GEMM, 0 if args.no_stream else 1)
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    if args.h2d:
        # Background H2D traffic like the link-bound decode step's expert streaming.
        hsrc = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        hdst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            for _ in range(200):
                hdst.copy_(hsrc, non_blocking=True)
    res = {}
    bf = torch.bfloat16
    # Expert FFN: 8 distinct experts (2.8 GB) so weights stream from HBM, not L2.
    if not args.only or args.only == "ffn":
        M = args.rows
        ws = [torch.randn(3 * d * f, dtype=bf, device=dev) * 0.02 for _ in range(E)]
        if args.kb:
            ws = [torch.cat([K.weights_kblock(w[: 2 * f * d].view(2 * f, d)).view(-1),
                             K.weights_kblock(w[2 * f * d:].view(d, f)).view(-1)]) for w in ws]
        kb = bool(args.kb)
        R = max(T * k, M)
        xp = torch.randn(R, d, dtype=bf, device=dev)
        y = torch.empty(R, d, dtype=bf, device=dev)
        h = torch.empty(max(M, 1), f, dtype=bf, device=dev)

        def ffn(i):
            w = ws[i % E]
            K.expert_ffn(xp, (i % E) * M % (R - M + 1), M, w[: 2 * f * d].view(2 * f, d),
                         w[2 * f * d:].view(d, f), y, h, kblocked=kb)
        t = timed(ffn, args.iters, st)
        byt = 3 * d * f * 2 + M * (2 * d * 2 + 2 * f * 2)
        res["expert_ffn"] = {"M": M, "us": t * 1e6, "GBs": byt / t / 1e9, "TFLOPs": 6 * M * d * f / t / 1e12}
        t = timed_graph(ffn, 16)
        res["expert_ffn_graph"] = {"M": M, "us": t * 1e6, "GBs": byt / t / 1e9}
        S = K.expert_ffn_deferred_splits(M, d, f)
        if kb and S:
            ypart = torch.empty(S, R, d, dtype=torch.float32, device=dev)

            def ffn_def(i):
                w = ws[i % E]
                K.expert_ffn_deferred(xp, (i % E) * M % (R - M + 1), M, w[: 2 * f * d].view(2 * f, d),
                                      w[2 * f * d:].view(d, f), ypart, h, S)
            t = timed_graph(ffn_def, 16)
            dump_trace("down_deferred")
            res["expert_ffn_deferred_graph"] = {"M": M, "splits": S, "us": t * 1e6, "GBs": byt / t / 1e9}
            if R >= E * M:
                # One layer block as the engine runs it at decode: 8 experts'
                # deferred FFNs, then the combine summing their split partials.
                Tt = R // k
                pos_b = torch.randperm(R, device=dev).to(torch.int32)
                wt_b = torch.rand(Tt, k, device=dev)
                res_b = torch.randn(Tt, d, dtype=bf, device=dev)
                out_b = torch.empty_like(res_b)

                def block(i):
                    for e in range(E):
                        w = ws[e]
                        K.expert_ffn_deferred(xp, e * M, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f),
                                              ypart, h, S)
                    K.combine_deferred(ypart, S, pos_b, wt_b, res_b, out=out_b)
                t = timed_graph(block, 4)
                res["block_8ffn_deferred_combine"] = {"M": M, "us": t * 1e6, "us_per_ffn": t * 1e6 / E}
            del ypart

        def g1(i):
            w = ws[i % E]
            K.gemm(xp, w[: 2 * f * d].view(2 * f, d), c=h, epilogue=2, row_offset=0, m=M, kblocked=kb)
        t = timed(g1, args.iters, st)
        dump_trace("gemm_swiglu")
        res["gemm_swiglu"] = {"M": M, "us": t * 1e6, "GBs": (2 * d * f * 2) / t / 1e9}
        t = timed_graph(g1, 16)
        res["gemm_swiglu_graph"] = {"M": M, "us": t * 1e6, "GBs": (2 * d * f * 2) / t / 1e9}

        def g2(i):
            w = ws[i % E]
            K.gemm(h, w[2 * f * d:].view(d, f), c=y[:M], m=M, kblocked=kb)
        t = timed(g2, args.iters, st)
        dump_trace("gemm_down")
        res["gemm_down"] = {"M": M, "us": t * 1e6, "GBs": (d * f * 2) / t / 1e9}
        t = timed_graph(g2, 16)
        res["gemm_down_graph"] = {"M": M, "us": t * 1e6, "GBs": (d * f * 2) / t / 1e9}
        del ws
    if not args.only or args.only == "attn":
        width = (Hq + 2 * Hkv) * hd
        wqkv = [torch.randn(width, d, dtype=bf, device=dev) * 0.02 for _ in range(4)]
        x = torch.randn(bs, d, dtype=bf, device=dev)
        qkv = torch.empty(bs, width, dtype=bf, device=dev)
        t = timed(lambda i: K.gemm(x, wqkv[i % 4], c=qkv), args.iters, st)
        res["gemm_qkv_M64"] = {"us": t * 1e6, "GBs": width * d * 2 / t / 1e9}
        dump_trace("qkv")
        wo = [torch.randn(d, Hq * hd, dtype=bf, device=dev) * 0.02 for _ in range(4)]
        ao = torch.randn(bs, Hq * hd, dtype=bf, device=dev)
        hres = torch.randn(bs, d, dtype=bf, device=dev)
        t = timed(lambda i: K.gemm(ao, wo[i % 4], c=hres, residual=hres, epilogue=1), args.iters, st)
        dump_trace("o_proj")
        res["gemm_oproj_M64"] = {"us": t * 1e6, "GBs": d * Hq * hd * 2 / t / 1e9}
        cap = 260
        kc = torch.randn(T * cap * Hkv * hd, dtype=bf, device=dev)
        vc = torch.randn_like(kc)
        pos = torch.full((bs,), 600, dtype=torch.int32, device=dev)
        seq = torch.arange(bs, dtype=torch.int32, device=dev)
        out = torch.empty(bs, Hq * hd, dtype=bf, device=dev)

        def att(i):
            K.attn_decode(qkv, width, pos, seq + (i % n) * bs, Hq, Hkv, hd, kc, vc, cap, 4, hd ** -0.5, out)
        t = timed(att, args.iters, st)
        res["attn_decode_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}

        seqs = [seq + j * bs for j in range(n)]

        def att2(i):
            K.attn_decode_split(qkv, width, pos, seqs[i % n], Hq, Hkv, hd, kc, vc, cap, 4, hd ** -0.5, out)
        t = timed(att2, args.iters, st)
        res["attn_decode_split_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}
        dump_trace("attn_decode_mma")
        t = timed_graph(att2, 20)
        res["attn_decode_mma_graph_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}
        K.tune(K.TUNE_DECODE_MMA, 0)
        t = timed_graph(att2, 20)
        res["attn_decode_cudacore_graph_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}
        K.tune(K.TUNE_DECODE_MMA, 1)
        K.tune(K.TUNE_DECODE_MMA, 2)
        t = timed(att2, args.iters, st)
        res["attn_decode_mma_loadonly_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}
        K.tune(K.TUNE_DECODE_MMA, 0)
        t = timed(att2, args.iters, st)
        K.tune(K.TUNE_DECODE_MMA, 1)
        res["attn_decode_split_cudacore_b64"] = {"us": t * 1e6, "GBs": bs * cap * Hkv * hd * 2 * 2 / t / 1e9}
    if args.only == "attnop":
        # The whole decode attention op as the engine issues it (rmsnorm, QKV
        # GEMM, RoPE + KV append, decode attention, o-proj with the residual
        # add), 8 batches x 4 layers with distinct weights and KV, one CUDA
        # graph; variants: o-proj through the weight-streaming GEMM, PDL off.
        width = (Hq + 2 * Hkv) * hd
        L4 = 4
        wqkv = [torch.randn(width, d, dtype=bf, device=dev) * 0.02 for _ in range(L4)]
        wo = [torch.randn(d, Hq * hd, dtype=bf, device=dev) * 0.02 for _ in range(L4)]
        nw = torch.ones(d, dtype=bf, device=dev)
        cap = 260
        kcs = [torch.randn(T * cap * Hkv * hd, dtype=bf, device=dev) for _ in range(L4)]
        vcs = [torch.randn(T * cap * Hkv * hd, dtype=bf, device=dev) for _ in range(L4)]
        h = torch.randn(T, d, dtype=bf, device=dev)
        xa = torch.empty(bs, d, dtype=bf, device=dev)
        qkv = torch.empty(bs, width, dtype=bf, device=dev)
        ao = torch.empty(bs, Hq * hd, dtype=bf, device=dev)
        pos = torch.full((bs,), 600, dtype=torch.int32, device=dev)
        seqs = [torch.arange(bs, dtype=torch.int32, device=dev) + j * bs for j in range(n)]

        def op(i):
            l, b = (i // n) % L4, i % n
            hb = h[b * bs:(b + 1) * bs]
            K.rmsnorm(hb, nw, out=xa)
            K.gemm(xa, wqkv[l], c=qkv)
            K.rope_kv_append(qkv, Hq, Hkv, hd, pos, seqs[b], 1e6, kcs[l], vcs[l], cap, 4)
            K.attn_decode_split(qkv, width, pos, seqs[b], Hq, Hkv, hd, kcs[l], vcs[l], cap, 4, hd ** -0.5, ao)
            K.gemm(ao, wo[l], c=hb, residual=hb, epilogue=1)
        per = 8 * L4
        tab = torch.empty(bs, hd // 2, 2, dtype=torch.float32, device=dev)

        def op_fused(i):
            # As the engine issues decode: RMSNorm + RoPE table, QKV GEMM with
            # the RoPE / KV-append epilogue, attention, o-proj.
            l, b = (i // n) % L4, i % n
            hb = h[b * bs:(b + 1) * bs]
            K.rmsnorm_rope_table(hb, nw, pos, 1e6, hd, out=xa, table=tab)
            assert K.qkv_rope(xa, wqkv[l], Hq, Hkv, hd, tab, pos, seqs[b], kcs[l], vcs[l], cap, 4, c=qkv) is not None
            K.attn_decode_split(qkv, width, pos, seqs[b], Hq, Hkv, hd, kcs[l], vcs[l], cap, 4, hd ** -0.5, ao)
            K.gemm(ao, wo[l], c=hb, residual=hb, epilogue=1)
        res["attn_op_b64_fused_rope"] = {"us": timed_graph(op_fused, per) * 1e6}
        Sq = K.gemm_deferred_splits(bs, width, d)
        if Sq:
            qpart = torch.empty(Sq, bs, width, dtype=torch.float32, device=dev)

            def op_defer(i):
                # As the engine issues decode: QKV splits left as fp32 partials,
                # summed by the RoPE / KV-append kernel.
                l, b = (i // n) % L4, i % n
                hb = h[b * bs:(b + 1) * bs]
                K.rmsnorm(hb, nw, out=xa)
                K.gemm_deferred(xa, wqkv[l], qpart, Sq)
                K.rope_kv_append_deferred(qpart, Sq, qkv, Hq, Hkv, hd, pos, seqs[b], 1e6, kcs[l], vcs[l], cap, 4)
                K.attn_decode_split(qkv, width, pos, seqs[b], Hq, Hkv, hd, kcs[l], vcs[l], cap, 4, hd ** -0.5, ao)
                K.gemm(ao, wo[l], c=hb, residual=hb, epilogue=1)
            res["attn_op_b64_deferred_qkv"] = {"us": timed_graph(op_defer, per) * 1e6, "splits": Sq}
            res["attn_op_part_qkv_deferred"] = {"us": timed_graph(
                lambda i: K.gemm_deferred(xa, wqkv[(i // n) % L4], qpart, Sq), per) * 1e6}

        def op_keep(i):
            # The layer's projection weights kept in L2 (evict-last) for all
            # but its last batch, which reads them evict-first.
            K.tune(K.TUNE_STREAM_HINT, 2 if i % n < n - 1 else 1)
            op(i)
            K.tune(K.TUNE_STREAM_HINT, 1)
        t = timed_graph(op_keep, per)
        res["attn_op_b64_l2keep"] = {"us": t * 1e6}
        t = timed_graph(op, per)
        res["attn_op_b64"] = {"us": t * 1e6, "floor_us": (width * d * 2 + d * Hq * hd * 2 + bs * cap * Hkv * hd * 4) / 6.5e6}
        K.tune(K.TUNE_STREAM_GEMM, 2)
        t = timed_graph(op, per)
        res["attn_op_b64_oproj_stream"] = {"us": t * 1e6}
        K.tune(K.TUNE_STREAM_GEMM, 1)
        K.tune(K.TUNE_PDL, 0)
        t = timed_graph(op, per)
        res["attn_op_b64_no_pdl"] = {"us": t * 1e6}
        K.tune(K.TUNE_PDL, 1)
        K.tune(K.TUNE_STREAM_EVEN_SPLIT, 2)
        t = timed_graph(op, per)
        res["attn_op_b64_near_even"] = {"us": t * 1e6}
        res["attn_op_part_qkv_near_even"] = {"us": timed_graph(lambda i: K.gemm(xa, wqkv[(i // n) % L4], c=qkv), per) * 1e6}
        K.tune(K.TUNE_STREAM_GEMM, 2)
        res["attn_op_part_oproj_stream_near_even"] = {"us": timed_graph(
            lambda i: K.gemm(ao, wo[(i // n) % L4], c=h[(i % n) * bs:(i % n + 1) * bs],
                             residual=h[(i % n) * bs:(i % n + 1) * bs], epilogue=1), per) * 1e6}
        K.tune(K.TUNE_STREAM_GEMM, 1)
        K.tune(K.TUNE_STREAM_EVEN_SPLIT, 2)
        for nm, fn in (("rmsnorm", lambda i: K.rmsnorm(h[(i % n) * bs:(i % n + 1) * bs], nw, out=xa)),
                       ("qkv", lambda i: K.gemm(xa, wqkv[(i // n) % L4], c=qkv)),
                       ("rope", lambda i: K.rope_kv_append(qkv, Hq, Hkv, hd, pos, seqs[i % n], 1e6, kcs[(i // n) % L4],
                                                           vcs[(i // n) % L4], cap, 4)),
                       ("attn", lambda i: K.attn_decode_split(qkv, width, pos, seqs[i % n], Hq, Hkv, hd, kcs[(i // n) % L4],
                                                              vcs[(i // n) % L4], cap, 4, hd ** -0.5, ao)),
                       ("oproj", lambda i: K.gemm(ao, wo[(i // n) % L4], c=h[(i % n) * bs:(i % n + 1) * bs],
                                                  residual=h[(i % n) * bs:(i % n + 1) * bs], epilogue=1))):
            res["attn_op_part_" + nm] = {"us": timed_graph(fn, per) * 1e6}
        K.tune(K.TUNE_STREAM_GEMM, 2)
        res["attn_op_part_oproj_stream"] = {"us": timed_graph(
            lambda i: K.gemm(ao, wo[(i // n) % L4], c=h[(i % n) * bs:(i % n + 1) * bs],
                             residual=h[(i % n) * bs:(i % n + 1) * bs], epilogue=1), per) * 1e6}
        K.tune(K.TUNE_STREAM_GEMM, 1)
    if not args.only or args.only == "route":
        h = torch.randn(T, d, dtype=bf, device=dev)
        nw = torch.ones(d, dtype=bf, device=dev)
        wg = torch.randn(E, d, dtype=bf, device=dev) * 0.02
        x2 = torch.empty_like(h)
        t = timed_graph(lambda i: K.gate_topk(h[:bs], nw, wg, k, x2=x2[:bs]), args.iters)
        res["gate_topk_b64"] = {"us": t * 1e6}
        _, idx, wt = K.gate_topk(h, nw, wg, k, x2=x2)
        t = timed_graph(lambda i: K.permute(idx, E, x2=x2), args.iters)
        res["permute_T512"] = {"us": t * 1e6, "GBs": (T * d * 2 + T * k * d * 2) / t / 1e9}
        _, _, p, _, xp = K.permute(idx, E, x2=x2)
        t = timed_graph(lambda i: K.combine(xp, p, wt, h, out=x2), args.iters)
        res["combine_T512"] = {"us": t * 1e6, "GBs": (k * T * d * 2 + 2 * T * d * 2) / t / 1e9}
        ypart = torch.randn(4, T * k, d, dtype=torch.float32, device=dev)
        t = timed_graph(lambda i: K.combine_deferred(ypart, 4, p, wt, h, out=x2), args.iters)
        res["combine_deferred4_T512"] = {"us": t * 1e6, "GBs": (4 * k * T * d * 4 + 2 * T * d * 2) / t / 1e9}
        del ypart
        t = timed_graph(lambda i: K.rmsnorm(h[:bs], nw, out=x2[:bs]), args.iters)
        res["rmsnorm_b64"] = {"us": t * 1e6, "GBs": 2 * bs * d * 2 / t / 1e9}
        # prefill-sized group: bs 32 x n 8 x 512 tokens
        TP = 32 * 8 * 512
        hp = torch.randn(TP, d, dtype=bf, device=dev)
        x2p = torch.empty_like(hp)
        _, idxp, wtp = K.gate_topk(hp, nw, wg, k, x2=x2p)
        t = timed(lambda i: K.permute(idxp, E, x2=x2p), max(2, args.iters // 4), st)
        res["permute_T131072"] = {"us": t * 1e6, "GBs": (TP * d * 2 + TP * k * d * 2) / t / 1e9}
        _, _, pp, _, xpp = K.permute(idxp, E, x2=x2p)
        t = timed(lambda i: K.combine(xpp, pp, wtp, hp, out=x2p), max(2, args.iters // 4), st)
        res["combine_T131072"] = {"us": t * 1e6, "GBs": (k * TP * d * 2 + 2 * TP * d * 2) / t / 1e9}
        del hp, x2p, xpp
    print(json.dumps(res, indent=1))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
