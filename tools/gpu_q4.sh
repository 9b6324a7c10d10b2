timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "prefill" 2>&1 | tail -2
for tc in 1 2; do echo "tc=$tc"; TC=$tc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_prefill_tc" -s 1 -c 2 python tools/prefill_attn_probe.py 2>&1 | grep -E "gpu__time" | cut -c1-70; done
