"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_r01.ncu-rep --out profiles/r01_ncu_summary.md
"""
import argparse
import collections
import csv
import io
import json
import subprocess

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(unit, v)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += to_us(r[vi], r[ui])
    return agg


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")}
        for w in WANT:
            if w in hdr:
                d[w] = r[hdr.index(w)] + (" " + units[hdr.index(w)] if units[hdr.index(w)] else "")
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", default="")
    ap.add_argument("--rep", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare shares)",
                  "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
        lines += ["", f"total: {sum(v[0] for v in agg.values())} launches, {tot:.1f} us", ""]
    if a.rep:
        lines += ["## --set full (per launch)", "", "```", json.dumps(full(a.rep), indent=1), "```", ""]
    open(a.out, "w").write("\n".join(lines))
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
