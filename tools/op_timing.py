"""Per-op durations of the engine's expert computes in a bench-shaped decode
run (timeline_csv + schedule), to compare in-step FFN time with the
microbenchmark. python tools/op_timing.py [--steps 2]"""
import argparse
import csv
import io
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_06888_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--hbm-cap", type=float, default=24e9)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--trace", action="store_true", help="per-CTA phase trace of the step's last streaming GEMM")
    ap.add_argument("--tune", action="append", default=[], help="kernel knob=value (kl_tune), repeatable")
    a = ap.parse_args()
    from paper_2502_06888_b200 import kernels as K
    K.tune(K.TUNE_PDL, a.pdl)
    for kv in a.tune:
        k, v = kv.split("=")
        K.tune(int(k), int(v))
    if a.trace:
        K.tune(99, 128)
    ns = argparse.Namespace(model="mixtral-8x7b", batch_size=64, n_batches=8, prompt_len=512, hbm_cap=a.hbm_cap,
                            host_distinct_layers=4, warmup=1, steps=a.steps)
    eng = Engine(bench.engine_config(ns, 0, 1))
    eng.fill_kv_synthetic(512)
    eng.step(1, None, want_next=False)
    eng.reset_log()
    for s in range(a.steps):
        eng.step(2 + s, None, want_next=False)
    if a.trace:
        import ctypes
        buf = (ctypes.c_ulonglong * (256 * 12))()
        K._lib.kl_stream_trace(buf, 256)
        tr = np.array(buf, dtype=np.float64).reshape(256, 12)[:148]
        t0 = tr[:, 0][tr[:, 0] > 0].min()
        rel = (tr - t0) / 1e3
        rel[tr == 0] = np.nan
        names = ["start", "mma0", "mma_end", "epi_last", "flags_ok", "landed", "sums_done", "end", "contrib0", "published"]
        print("in-step trace of the last streaming GEMM (us from first CTA start)")
        for i, nm in enumerate(names):
            col = rel[:, i]
            if np.all(np.isnan(col)):
                continue
            print(f"  {nm:10s} med {np.nanmedian(col):7.2f}  min {np.nanmin(col):7.2f}  max {np.nanmax(col):7.2f}")
    tl = eng.report("timeline_csv")["text"]
    rows = list(csv.DictReader(io.StringIO(tl)))
    print("columns:", list(rows[0].keys()))
    by = {}
    for r in rows:
        k = r.get("kind") or r.get("op_kind")
        dur = (int(r["end_ps"]) - int(r["start_ps"])) / 1e6 if "end_ps" in r else None
        by.setdefault(k, []).append((dur, int(r.get("tokens", 0) or 0)))
    for k, v in by.items():
        d = np.array([x[0] for x in v if x[0] is not None])
        t = np.array([x[1] for x in v])
        if len(d):
            print(f"{k:20s} n={len(d):5d} mean {d.mean():9.1f} us  med {np.median(d):9.1f}  p90 {np.percentile(d, 90):9.1f}"
                  f"  tokens mean {t.mean():.1f} max {t.max()}")
    ex = [(x[0], x[1]) for x in by.get("compute_expert", [])]
    if ex:
        ex.sort(key=lambda z: z[1])
        for lo, hi in [(0, 64), (64, 128), (128, 160), (160, 256), (256, 10**9)]:
            sel = [d for d, t in ex if lo < t <= hi]
            if sel:
                print(f"  rows ({lo},{hi}]: n={len(sel)} mean {np.mean(sel):.1f} us")
    # Expert ops split by whether they waited for their load: gap to the
    # previous compute-stream op's end (small = weights were already there).
    comp = sorted([r for r in rows if r["stream"] == "compute"], key=lambda r: int(r["start_ps"]))
    waited, ready = [], []
    for prev, r in zip(comp, comp[1:]):
        if r["kind"] != "compute_expert":
            continue
        gap = (int(r["start_ps"]) - int(prev["end_ps"])) / 1e6
        dur = (int(r["end_ps"]) - int(r["start_ps"])) / 1e6
        (waited if gap > 5.0 else ready).append((dur, gap, prev["kind"]))
    for name, v in (("waited for load", waited), ("load already done", ready)):
        if v:
            d = np.array([x[0] for x in v])
            print(f"  {name:18s} n={len(d):4d} dur mean {d.mean():.1f} med {np.median(d):.1f} us;"
                  f" gap med {np.median([x[1] for x in v]):.1f} us")
    eng.close()


if __name__ == "__main__":
    main()
