"""One decode step of the bench workload bracketed by cudaProfilerStart/Stop,
for an ncu launch list of exactly that step:

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/step_profile.py [--resident]

--resident: the all-resident (compute-exposed) configuration of bench.py's
`resident` key (HBM cap 140e9 B); default: the headline (24e9 B cap,
experts streamed).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_06888_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--resident", action="store_true")
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    ns = argparse.Namespace(model="mixtral-8x7b", batch_size=64, n_batches=8, prompt_len=512,
                            hbm_cap=140e9 if a.resident else 24e9, host_distinct_layers=0 if a.resident else 4,
                            warmup=a.warmup, steps=1)
    eng = Engine(bench.engine_config(ns, 0, 1))
    eng.fill_kv_synthetic(512)
    step = 1
    for _ in range(a.warmup):
        eng.step(step, None, want_next=False)
        step += 1
    import torch
    rt = torch.cuda.cudart()
    rt.cudaProfilerStart()
    _, ms = eng.step(step, None, want_next=False)
    rt.cudaProfilerStop()
    print(f"step {step}: {ms:.2f} ms", file=sys.stderr)
    eng.close()


if __name__ == "__main__":
    main()
