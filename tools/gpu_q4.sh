mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "q4 or stream or gemm or ffn" 2>&1 | tail -2
run() { echo "== $*"; timeout 120 python "$@" --only ffn --iters 30 2>&1 | grep -E '"us"' | tr -d '\n'; echo; }
run prev_build/tools/profile_kernels.py --rows 128
run tools/profile_kernels.py --rows 128
