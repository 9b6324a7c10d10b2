"""Where do the in-step expert-op microseconds go? Every case queues its whole
sequence behind a 1-thread kernel that spins on a host-mapped flag
(kl_debug_spin_flag), so host launch latency is excluded; events time the
FFN (kl_expert_ffn at Mixtral-8x7B shape, M rows):
  cold        : spin -> a -> FFN -> b                (GPU idle before, no PDL overlap)
  b2b_events  : spin -> a0 FFN b0 a1 FFN b1 ...       (event records between ops, no waits)
  b2b_plain   : spin -> a FFN FFN ... FFN b           (per FFN, no events between)
  xwait_small : copy stream: spin -> 1 MB H2D -> ev;  compute: wait ev -> a -> FFN -> b
  xwait_big   : copy stream: spin -> expert H2D -> ev; compute: wait ev -> a -> FFN -> b
  xwait_chain : compute has a prior FFN running; the next FFN waits for an
                expert copy that lands after it
  pipeline    : experts streamed back to back into a 4-slot ring, each FFN
                waits for its own copy (the next copy in flight meanwhile):
                the engine's link-bound in-step shape
python tools/op_latency_probe.py"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402
from paper_2502_06888_b200 import load_native  # noqa: E402

_lib = load_native()
_lib.kl_debug_spin_flag.argtypes = [C.c_void_p, C.c_void_p]
_lib.kl_debug_spin_flag.restype = C.c_int


def main():
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    d, f, M = 4096, 14336, int(os.environ.get("M", "128"))
    ne = 3 * d * f
    host = torch.empty(ne, dtype=bf, pin_memory=True)
    small = torch.empty(512 * 1024, dtype=bf, pin_memory=True)
    slots = [torch.empty(ne, dtype=bf, device=dev) for _ in range(4)]
    for s in slots:
        K.fill_normal(s, 7, 0.02)
    dsmall = torch.empty_like(small, device=dev)
    xp = torch.randn(M, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(M, f, dtype=bf, device=dev)
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream()
    flag = torch.zeros(4, dtype=torch.int32, pin_memory=True)

    def spin(stream):
        flag[0] = 0
        assert _lib.kl_debug_spin_flag(C.c_void_p(flag.data_ptr()), C.c_void_p(stream.cuda_stream)) == 0

    def release():
        flag[0] = 1

    def ffn(w):
        K.expert_ffn(xp, 0, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h, stream=cs.cuda_stream)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def med(xs):
        xs = sorted(xs)
        return round(xs[len(xs) // 2], 1)

    for i in range(6):
        ffn(slots[i % 4])
    torch.cuda.synchronize()
    reps = 7
    res = {"M": M}

    out = []
    for r in range(reps):
        spin(cs)
        a, b = ev(), ev()
        a.record(cs)
        ffn(slots[r % 4])
        b.record(cs)
        release()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    res["cold"] = med(out)

    out = []
    for r in range(reps):
        spin(cs)
        evs = []
        for i in range(8):
            a, b = ev(), ev()
            a.record(cs)
            ffn(slots[i % 4])
            b.record(cs)
            evs.append((a, b))
        release()
        torch.cuda.synchronize()
        out += [a.elapsed_time(b) * 1e3 for a, b in evs[1:]]
    res["b2b_events"] = med(out)

    out = []
    for r in range(reps):
        spin(cs)
        a, b = ev(), ev()
        a.record(cs)
        for i in range(8):
            ffn(slots[i % 4])
        b.record(cs)
        release()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3 / 8)
    res["b2b_plain"] = med(out)

    # the engine's K-blocked expert layout (kl_expert_ffn_kb), back to back
    kbs = []
    for sl in slots[:3]:
        t = torch.empty_like(sl)
        t[: 2 * f * d].view(2 * f, d).copy_(K.weights_kblock(sl[: 2 * f * d].view(2 * f, d)))
        t[2 * f * d:].view(d, f).copy_(K.weights_kblock(sl[2 * f * d:].view(d, f)))
        kbs.append(t)
    out = []
    for r in range(reps):
        spin(cs)
        a, b = ev(), ev()
        a.record(cs)
        for i in range(9):
            w = kbs[i % 3]
            K.expert_ffn(xp, 0, M, w[: 2 * f * d].view(2 * f, d), w[2 * f * d:].view(d, f), y, h,
                         stream=cs.cuda_stream, kblocked=True)
        b.record(cs)
        release()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3 / 9)
    res["b2b_plain_kblocked"] = med(out)
    del kbs

    def xwait(big, chain=False):
        out = []
        for r in range(reps):
            w = slots[r % 4]
            spin(ls)
            if chain:
                # a prior FFN on the compute stream, started right away
                ffn(slots[(r + 1) % 4])
            with torch.cuda.stream(ls):
                if big:
                    w.copy_(host, non_blocking=True)
                else:
                    dsmall.copy_(small, non_blocking=True)
            loaded = torch.cuda.Event()
            loaded.record(ls)
            cs.wait_event(loaded)
            a, b = ev(), ev()
            a.record(cs)
            ffn(w)
            b.record(cs)
            release()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b) * 1e3)
        return med(out)

    def pipeline(nslots=4, iters=10, chunks=1, serial=False, other=False):
        """The in-step shape: the copy stream streams experts back to back
        into a slot ring; each FFN waits for its own expert, so the next copy
        is always in flight while an FFN runs."""
        out = []
        for r in range(2):
            spin(ls)
            done = [None] * iters
            evs = []
            for i in range(iters):
                w = slots[i % nslots]
                if i >= nslots:
                    ls.wait_event(done[i - nslots])
                if serial and i >= 1:
                    ls.wait_event(done[i - 1])  # no copy in flight during an FFN
                with torch.cuda.stream(ls):
                    step = ne // chunks
                    for c in range(chunks):
                        w[c * step:(c + 1) * step if c < chunks - 1 else ne].copy_(
                            host[c * step:(c + 1) * step if c < chunks - 1 else ne], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(ls)
                cs.wait_event(loaded)
                a, b = ev(), ev()
                a.record(cs)
                ffn(slots[(i + 2) % nslots] if other else w)  # other: a slot not written recently
                b.record(cs)
                done[i] = torch.cuda.Event()
                done[i].record(cs)
                evs.append((a, b))
            release()
            torch.cuda.synchronize()
            out += [a.elapsed_time(b) * 1e3 for a, b in evs[1:]]
        return med(out)

    res["pipeline"] = pipeline()
    # Host buffer backed by transparent huge pages (2 MB), registered with
    # cudaHostRegister: fewer sysmem translations for the copy engine.
    import mmap
    nbytes = ne * 2
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        mm.madvise(mmap.MADV_HUGEPAGE)
    except Exception:
        pass
    huge = torch.frombuffer(mm, dtype=torch.uint8)
    off = (-huge.data_ptr()) % (2 << 20)
    huge = huge[off:off + nbytes]
    huge.fill_(1)
    rc = torch.cuda.cudart().cudaHostRegister(huge.data_ptr(), nbytes, 0)
    res["host_register_rc"] = int(rc)
    try:
        with open("/sys/kernel/mm/transparent_hugepage/enabled") as fh:
            res["thp"] = fh.read().strip()
        with open("/proc/meminfo") as fh:
            res["anon_huge_kb"] = [l for l in fh if l.startswith("AnonHugePages")][0].split()[1]
    except OSError:
        pass
    saved = host
    host = huge.view(torch.bfloat16)
    res["pipeline_thp_host"] = pipeline()
    host = saved
    res["pipeline_8chunks"] = pipeline(chunks=8)

    def interfere(kind, iters=8):
        """FFNs back to back (events around each) while the copy stream runs
        a long transfer of one kind."""
        big_h = torch.empty(ne, dtype=bf, pin_memory=True)
        d16 = torch.empty(8 << 20, dtype=bf, device=dev)
        h16 = torch.empty(8 << 20, dtype=bf, pin_memory=True)
        out = []
        for r in range(2):
            spin(cs)
            with torch.cuda.stream(ls):
                for _ in range(3):
                    if kind == "h2d":
                        slots[3].copy_(host, non_blocking=True)
                    elif kind == "d2h":
                        big_h.copy_(slots[3], non_blocking=True)
                    elif kind == "h2d_16mb_repeat":
                        for _ in range(22):
                            d16.copy_(h16, non_blocking=True)
                    elif kind == "d2d":
                        slots[3][: ne // 8].copy_(slots[2][: ne // 8], non_blocking=True)
            evs = []
            for i in range(iters):
                a, b = ev(), ev()
                a.record(cs)
                ffn(slots[i % 3])
                b.record(cs)
                evs.append((a, b))
            release()
            torch.cuda.synchronize()
            out += [a.elapsed_time(b) * 1e3 for a, b in evs[1:]]
        return med(out)

    for kind in ("h2d", "d2h", "h2d_16mb_repeat", "d2d"):
        res["b2b_events_with_" + kind] = interfere(kind)

    # SM-driven zero-copy H2D (tools/zc): its own bandwidth, and the FFN with it in flight.
    zc = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "zc", "libzc.so"))
    zc.zc_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]
    for ctas, thr in ((16, 512), (32, 512), (64, 256)):
        a, b = ev(), ev()
        a.record(ls)
        assert zc.zc_copy(slots[3].data_ptr(), host.data_ptr(), ne * 2, ctas, thr, ls.cuda_stream) == 0
        b.record(ls)
        torch.cuda.synchronize()
        res[f"zc_gbs_{ctas}x{thr}"] = round(ne * 2 / (a.elapsed_time(b) / 1e3) / 1e9, 1)
        out = []
        for r in range(2):
            spin(cs)
            for _ in range(2):
                zc.zc_copy(slots[3].data_ptr(), host.data_ptr(), ne * 2, ctas, thr, ls.cuda_stream)
            evs = []
            for i in range(8):
                a, b = ev(), ev()
                a.record(cs)
                ffn(slots[i % 3])
                b.record(cs)
                evs.append((a, b))
            release()
            torch.cuda.synchronize()
            out += [a.elapsed_time(b) * 1e3 for a, b in evs[1:]]
        res[f"b2b_events_with_zc_{ctas}x{thr}"] = med(out)
    res["pipeline_serial"] = pipeline(serial=True)
    res["pipeline_other_slot"] = pipeline(other=True)
    res["xwait_small"] = xwait(False)
    res["xwait_big"] = xwait(True)
    res["xwait_chain"] = xwait(True, chain=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
