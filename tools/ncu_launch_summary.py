"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel launches, total time and share. python tools/ncu_launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("kl::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    print(f"\ntotal: {sum(v[0] for v in agg.values())} launches, {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
