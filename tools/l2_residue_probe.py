"""In-step shape of the expert FFN without timed events: the copy stream
streams experts back to back into a 4-slot ring (untimed events), the compute
stream runs each FFN after its own copy, bracketed by device timestamps
(kl_stamp, as the engine does). Does reading weights the copy engine has just
written (partly still dirty in L2) slow the FFN, and does the copy order of
W13 / W2 matter?

    python tools/l2_residue_probe.py  ->  JSON (median us per FFN per case)
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
n13 = 2 * f * d


def main():
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    lib = K._lib
    lib.kl_stamp.argtypes = [C.c_void_p, C.c_void_p]
    lib.kl_stamp.restype = C.c_int
    hosts = []
    for e in range(2):
        w = torch.empty(ne, dtype=bf, device=dev)
        K.fill_normal(w, 31 + e, 0.02)
        kb = torch.empty_like(w)
        kb[:n13].view(2 * f, d).copy_(K.weights_kblock(w[:n13].view(2 * f, d)))
        kb[n13:].view(d, f).copy_(K.weights_kblock(w[n13:].view(d, f)))
        hosts.append(kb.cpu().pin_memory())
        del w, kb
    slots = [torch.empty(ne, dtype=bf, device=dev) for _ in range(4)]
    others = [torch.empty(ne, dtype=bf, device=dev) for _ in range(2)]  # never written by the copies
    for o in others:
        K.fill_normal(o, 5, 0.02)
    xp = torch.randn(M, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(M, f, dtype=bf, device=dev)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
    stamps = torch.zeros(2 * 64, dtype=torch.int64, device=dev)

    def stamp(i, side):
        assert lib.kl_stamp(C.c_void_p(stamps.data_ptr() + 8 * (2 * i + side)), C.c_void_p(cs.cuda_stream)) == 0

    def ffn(w):
        K.expert_ffn(xp, 0, M, w[:n13].view(2 * f, d), w[n13:].view(d, f), y, h, stream=cs.cuda_stream,
                     kblocked=True)

    def run(case, n=12):
        done = []
        with torch.cuda.stream(ls):
            for i in range(n):
                w, src = slots[i % 4], hosts[i % 2]
                if i >= 4:
                    ls.wait_event(done[i - 4][1])  # slot free once its FFN ended
                if case == "w2_first":
                    w[n13:].copy_(src[n13:], non_blocking=True)
                    w[:n13].copy_(src[:n13], non_blocking=True)
                else:
                    w.copy_(src, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(ls)
                fin = torch.cuda.Event()
                with torch.cuda.stream(cs):
                    if case == "other_slot":
                        cs.wait_event(ev)
                        stamp(i, 0)
                        ffn(others[i % 2])  # weights the copy engine did not just write
                    else:
                        cs.wait_event(ev)
                        stamp(i, 0)
                        ffn(w)
                    stamp(i, 1)
                    fin.record(cs)
                done.append((ev, fin))
        torch.cuda.synchronize()
        t = stamps[: 2 * n].view(n, 2).cpu().double()
        us = sorted(((t[:, 1] - t[:, 0]) / 1e3).tolist()[2:])
        return us[len(us) // 2]

    res = {"M": M}
    for case in ("own_copy", "w2_first", "other_slot"):
        run(case, 6)
        res[case] = run(case)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
