timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "decode_attention" 2>&1 | tail -1
timeout 300 python tools/profile_kernels.py --only attn --iters 20 2>&1 | grep -A1 graph | grep -v GBs
