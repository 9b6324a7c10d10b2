mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "prefill" --durations=5 2>&1 | tail -15
timeout 600 python tools/prefill_run.py --bs 8 --n 8 --reps 2 2>&1 | tail -2
