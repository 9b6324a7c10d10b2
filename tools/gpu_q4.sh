mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "persistent or gemm or ffn" 2>&1 | tail -2
for r in 2048 8192 32768; do echo "== rows $r"; timeout 300 python tools/profile_kernels.py --only ffn --rows $r --iters 5 2>&1 | grep -A4 '"expert_ffn"\|"gemm_swiglu"\|"gemm_down"' | grep -E 'us|TFLOP'; done
echo "== rows 8192 non-persistent"; timeout 300 python tools/profile_kernels.py --only ffn --rows 8192 --iters 5 --persist 0 2>&1 | grep -A4 '"expert_ffn"' | grep -E 'us|TFLOP'
