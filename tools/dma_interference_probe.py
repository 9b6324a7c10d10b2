"""Does a concurrent pinned-host -> HBM copy slow the expert FFN, and under
which launch shapes? Every case records events on both streams so the copy's
overlap with the FFN window is checked, not assumed.

    python tools/dma_interference_probe.py  ->  one JSON object on stdout
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402

d, f, M = 4096, 14336, int(os.environ.get("M", "128"))
ne = 3 * d * f
dev = torch.device("cuda:0")
bf = torch.bfloat16


def main():
    E = 8
    ws = []
    for e in range(E):
        w = torch.empty(ne, dtype=bf, device=dev)
        K.fill_normal(w, 11 + e, 0.02)
        kb = torch.empty_like(w)
        kb[: 2 * f * d].view(2 * f, d).copy_(K.weights_kblock(w[: 2 * f * d].view(2 * f, d)))
        kb[2 * f * d:].view(d, f).copy_(K.weights_kblock(w[2 * f * d:].view(d, f)))
        ws.append(kb)
        del w
    xp = torch.randn(M, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(M, f, dtype=bf, device=dev)
    cs = torch.cuda.Stream()
    ls = torch.cuda.Stream()
    host = torch.empty(ne, dtype=bf, pin_memory=True)
    host1g = torch.empty(1 << 29, dtype=bf, pin_memory=True)
    dst = torch.empty(ne, dtype=bf, device=dev)
    dst1g = torch.empty(1 << 29, dtype=bf, device=dev)

    lib = K._lib
    lib.kl_stamp.argtypes = [C.c_void_p, C.c_void_p]
    lib.kl_stamp.restype = C.c_int
    stamps = torch.zeros(4 * 64, dtype=torch.int64, device=dev)

    def ffn(i, events=None):
        w = ws[i % E]
        if events is not None:
            events[0].record(cs)
        K.expert_ffn(xp, 0, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h,
                     stream=cs.cuda_stream, kblocked=True)
        if events is not None:
            events[1].record(cs)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n = 32
    for i in range(8):
        ffn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for i in range(n):
                ffn(i)
    torch.cuda.synchronize()

    def start_copy(kind, count):
        a, b = ev(), ev()
        with torch.cuda.stream(ls):
            a.record(ls)
            for _ in range(count):
                if kind == "h2d":
                    dst.copy_(host, non_blocking=True)
                elif kind == "h2d_1g":
                    dst1g.copy_(host1g, non_blocking=True)
                elif kind == "d2h":
                    host.copy_(dst, non_blocking=True)
            b.record(ls)
        return a, b

    def run(kind, mode):
        copy = None
        if kind:
            copy = start_copy(kind, 3 if kind != "h2d_1g" else 1)
        a, b = ev(), ev()
        per = []
        with torch.cuda.stream(cs):
            if copy is not None:
                cs.wait_event(copy[0])
            a.record(cs)
            if mode == "graph":
                g.replay()
            elif mode == "events":
                for i in range(n):
                    e2 = (ev(), ev())
                    ffn(i, e2)
                    per.append(e2)
            else:
                for i in range(n):
                    ffn(i)
            b.record(cs)
        torch.cuda.synchronize()
        out = {"us_per_ffn": a.elapsed_time(b) * 1e3 / n}
        if per:
            xs = sorted(x.elapsed_time(y_) * 1e3 for x, y_ in per)
            out["event_us_median"] = xs[len(xs) // 2]
        if copy is not None:
            ca, cb = copy
            out["copy_ms"] = ca.elapsed_time(cb)
            out["ffn_start_after_copy_start_ms"] = ca.elapsed_time(a)
            out["ffn_end_before_copy_end_ms"] = b.elapsed_time(cb)
            out["overlapped"] = out["ffn_end_before_copy_end_ms"] > 0
        return out

    def marked(kind, marker):
        """FFNs back to back with a marker pair (start, end) around each."""
        copy = start_copy(kind, 3) if kind else None
        a, b = ev(), ev()
        with torch.cuda.stream(cs):
            if copy is not None:
                cs.wait_event(copy[0])
            a.record(cs)
            for i in range(n):
                for side in (0, 1):
                    if side == 1:
                        ffn(i)
                    if marker == "timed_event":
                        torch.cuda.Event(enable_timing=True).record(cs)
                    elif marker == "untimed_event":
                        torch.cuda.Event(enable_timing=False).record(cs)
                    elif marker == "untimed_event_end_only" and side == 1:
                        torch.cuda.Event(enable_timing=False).record(cs)
                    elif marker == "timed_event_end_only" and side == 1:
                        torch.cuda.Event(enable_timing=True).record(cs)
                    elif marker == "stamp":
                        assert lib.kl_stamp(C.c_void_p(stamps.data_ptr() + 8 * (2 * i + side)), C.c_void_p(cs.cuda_stream)) == 0
            b.record(cs)
        torch.cuda.synchronize()
        out = {"us_per_ffn": a.elapsed_time(b) * 1e3 / n}
        if marker == "stamp":
            t = stamps[: 2 * n].view(n, 2).cpu().double()
            d_ = ((t[:, 1] - t[:, 0]) / 1e3).tolist()
            d_.sort()
            out["stamp_us_median"] = d_[len(d_) // 2]
        if copy is not None:
            out["overlapped"] = b.elapsed_time(copy[1]) > 0
        return out

    res = {"M": M}
    for marker in ("none", "timed_event", "untimed_event", "timed_event_end_only", "untimed_event_end_only", "stamp"):
        for kind in (None, "h2d", "d2h"):
            r = [marked(kind, marker) for _ in range(3)]
            r.sort(key=lambda z: z["us_per_ffn"])
            res[f"marker_{marker}_{kind or 'idle'}"] = r[1]
    for mode in ("graph", "eager", "events"):
        for kind in (None, "h2d", "h2d_1g", "d2h"):
            key = f"{mode}_{kind or 'idle'}"
            r = [run(kind, mode) for _ in range(3)]
            r.sort(key=lambda z: z["us_per_ffn"])
            res[key] = r[1]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
