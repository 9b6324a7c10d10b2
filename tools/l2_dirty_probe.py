"""Why is the expert FFN slower in-step than back-to-back? Hypothesis: the
expert's H2D copy leaves up to ~100 MB of its tail dirty in L2; the FFN's
first reads evict those lines (write-backs) before it reaches them again.
Times the FFN (CUDA events on its stream) after different preceding
conditions:
  after_copy_same   : H2D copy into the slot, sync, FFN on that slot
  after_copy_other  : H2D copy into another slot, sync, FFN on a slot not
                      recently written (L2 dirty with unrelated lines)
  after_clean       : FFN after a 256 MB read pass (L2 holds clean lines)
  after_copy_rev    : copy W2 first, then W13, sync, FFN on that slot
  copy_in_flight    : FFN on a loaded slot while the next H2D copy runs
  b2b               : back-to-back FFNs (graph-free), per call
python tools/l2_dirty_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    d, f, M = 4096, 14336, int(os.environ.get("M", "128"))
    ne = 3 * d * f
    host = torch.empty(ne, dtype=bf, pin_memory=True)
    host.view(torch.int16).random_(-2000, 2000)
    slots = [torch.empty(ne, dtype=bf, device=dev) for _ in range(3)]
    for s in slots:
        K.fill_normal(s, 7, 0.02)
    scratch = torch.empty(256 * 1024 * 1024 // 2, dtype=bf, device=dev)
    xp = torch.randn(M, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(M, f, dtype=bf, device=dev)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()

    def ffn(w):
        K.expert_ffn(xp, 0, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h, stream=cs.cuda_stream)

    def timed(w):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        ffn(w)
        b.record(cs)
        return a, b

    def med(xs):
        xs = sorted(xs)
        return round(xs[len(xs) // 2], 1)

    res = {}
    reps = 9
    # warm-up
    for i in range(4):
        ffn(slots[i % 3])
    torch.cuda.synchronize()

    def case(prep, slot):
        out = []
        for _ in range(reps):
            prep()
            torch.cuda.synchronize()
            a, b = timed(slots[slot])
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b) * 1e3)
        return med(out)

    def copy_into(i):
        with torch.cuda.stream(ls):
            slots[i].copy_(host, non_blocking=True)

    def copy_rev(i):
        with torch.cuda.stream(ls):
            slots[i][2 * f * d:].copy_(host[2 * f * d:], non_blocking=True)
            slots[i][: 2 * f * d].copy_(host[: 2 * f * d], non_blocking=True)

    def clean():
        with torch.cuda.stream(cs):
            scratch.add_(0)  # read + write 256 MB: the L2 ends up with scratch lines

    def clean_read():
        with torch.cuda.stream(cs):
            torch.sum(scratch.view(torch.int16).view(-1, 4096)[:, :1].float())

    res["after_copy_same"] = case(lambda: copy_into(0), 0)
    res["after_copy_other"] = case(lambda: copy_into(1), 0)
    res["after_clean_rw"] = case(clean, 0)
    res["after_copy_rev"] = case(lambda: copy_rev(0), 0)
    res["after_copy_then_clean"] = case(lambda: (copy_into(0), torch.cuda.synchronize(), clean()), 0)
    # FFN on slot 0 while the copy into slot 1 is in flight
    inflight = []
    for _ in range(reps):
        torch.cuda.synchronize()
        copy_into(1)
        a, b = timed(slots[0])
        torch.cuda.synchronize()
        inflight.append(a.elapsed_time(b) * 1e3)
    res["copy_in_flight"] = med(inflight)
    # realistic: copy into slot i, FFN on slot i as soon as copy done, next copy already started
    real = []
    for it in range(reps):
        torch.cuda.synchronize()
        i = it % 3
        copy_into(i)
        ev = torch.cuda.Event()
        ev.record(ls)
        copy_into((i + 1) % 3)
        cs.wait_event(ev)
        a, b = timed(slots[i])
        torch.cuda.synchronize()
        real.append(a.elapsed_time(b) * 1e3)
    res["pipelined_copy_then_ffn"] = med(real)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    for i in range(12):
        ffn(slots[i % 3])
    b.record(cs)
    torch.cuda.synchronize()
    res["b2b"] = round(a.elapsed_time(b) * 1e3 / 12, 1)
    res["M"] = M
    print(json.dumps(res))


if __name__ == "__main__":
    main()
