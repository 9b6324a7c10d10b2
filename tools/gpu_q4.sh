mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/prefill_run.py --bs 8 --n 8 --reps 1 2>&1 | tail -1 | cut -c1-600
