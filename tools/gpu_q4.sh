timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "prefill" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_prefill_tc" -c 3 python tools/prefill_run.py --bs 32 --n 8 --reps 1 2>&1 | grep -E "gpu__time" | cut -c1-70
