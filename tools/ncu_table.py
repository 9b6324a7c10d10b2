"""Per-kernel table from an ncu report: time, DRAM bytes, achieved DRAM
GB/s, grid, registers (python tools/ncu_table.py report.ncu-rep [regex])."""
import csv
import io
import re
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
     "launch__block_size", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {m: h.index(m) for m in M}
    name = h.index("Kernel Name")
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    print("| kernel | time us | DRAM read MB | DRAM write MB | GB/s | dram % peak | grid x block | regs |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        k = re.sub(r"\(.*", "", r[name]).replace("void ", "").replace("(anonymous namespace)::", "")
        if pat and not pat.search(k):
            continue
        t = float(r[col[M[0]]])
        if units[col[M[0]]] == "ns":
            t /= 1e3
        elif units[col[M[0]]] == "ms":
            t *= 1e3
        rd = float(r[col[M[1]]]) * scale.get(units[col[M[1]]], 1.0)
        wr = float(r[col[M[2]]]) * scale.get(units[col[M[2]]], 1.0)
        print(f"| {k[:60]} | {t:.2f} | {rd:.2f} | {wr:.2f} | {(rd + wr) / t * 1e3:.0f} | "
              f"{float(r[col[M[7]]]):.1f} | {r[col[M[3]]]} x {r[col[M[4]]]} | {r[col[M[5]]]} |")


if __name__ == "__main__":
    main()
