"""profiles/ncu_expert_ffn.json from an ncu --set full capture of one expert
FFN (tools/gpu_ffn_ncu.sh): DRAM read + write bytes of its two
weight-streaming GEMM launches (bench.py's roofline `traffic`).

    python tools/ncu_ffn_traffic.py gpurun_out/r02_ffn_full.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {m: h.index(m) for m in M if m in h}
    name = h.index("Kernel Name")
    kernels, total = [], 0.0
    for r in rows[2:]:
        k = {"kernel": r[name][:80]}
        for m, c in col.items():
            v = float(r[c].replace(",", ""))
            k[m] = v * SCALE.get(units[c], 1.0)
        total += k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        kernels.append(k)
    algo = 3 * 4096 * 14336 * 2 + 128 * (2 * 4096 * 2 + 2 * 14336 * 2)
    res = {"source": "ncu --set full --clock-control none, tools/gpu_ffn_ncu.sh (profile_kernels --only ffn, "
                     "K-blocked weights, M 128), round 2",
           "kernels_per_op": [k["kernel"] for k in kernels],
           "per_kernel": kernels,
           "dram_bytes_per_op": int(total),
           "algorithmic_bytes_per_op_at_M128": algo,
           "traffic_over_algorithmic": total / algo,
           "note": "dram read+write summed over the two weight-streaming GEMM launches of one compute_expert op; "
                   "ncu times are cold-cache and serialised"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_expert_ffn.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
