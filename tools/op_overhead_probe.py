"""In-step structure of a compute_expert op, emulated: a copy stream moves
the expert's weights H2D and records an event; the compute stream waits on
it, records start, runs the expert FFN, records end. Compares end - start
with the FFN alone, with and without the event records.
python tools/op_overhead_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    d, f, M = 4096, 14336, 128
    nb = 3 * d * f * 2
    host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    nslots = int(os.environ.get("SLOTS", "2"))
    slots = [torch.empty(3 * d * f, dtype=bf, device=dev) for _ in range(nslots)]
    for s in slots:
        K.fill_normal(s, 7, 0.02)
    xp = torch.randn(M, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(M, f, dtype=bf, device=dev)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()

    def ffn(w):
        K.expert_ffn(xp, 0, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h, stream=cs.cuda_stream)

    res = {}
    for variant in ("events", "no_start_event", "ffn_only_after_wait"):
        durs = []
        for it in range(24):
            w = slots[it % nslots]
            loaded = torch.cuda.Event()
            with torch.cuda.stream(ls):
                w.view(torch.uint8).copy_(host, non_blocking=True)
                loaded.record(ls)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cs.wait_event(loaded)
            if variant == "events":
                a.record(cs)
                ffn(w)
                b.record(cs)
            elif variant == "no_start_event":
                ffn(w)
                b.record(cs)
                a = loaded  # (not timed)
            else:
                ffn(w)
            torch.cuda.synchronize()
            if variant == "events" and it >= 2:
                durs.append(a.elapsed_time(b) * 1e3)
        if durs:
            durs.sort()
            res[variant] = round(durs[len(durs) // 2], 1)
    # the FFN alone, back to back, and once from idle
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        a.record(cs)
        for i in range(10):
            ffn(slots[i % 2])
        b.record(cs)
    torch.cuda.synchronize()
    res["ffn_back_to_back"] = round(a.elapsed_time(b) * 1e3 / 10, 1)
    idle = []
    for i in range(8):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            a.record(cs)
            ffn(slots[i % 2])
            b.record(cs)
        torch.cuda.synchronize()
        idle.append(a.elapsed_time(b) * 1e3)
    idle.sort()
    res["ffn_from_idle_host_enqueued"] = round(idle[len(idle) // 2], 1)
    print(res)


if __name__ == "__main__":
    main()
