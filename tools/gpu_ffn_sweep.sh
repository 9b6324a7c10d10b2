mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu 2>&1 | tail -2
run() { echo "== $*"; timeout 120 python tools/profile_kernels.py --only ffn --iters 20 "$@" 2>&1 | grep -E '"us"' | tr -d '\n'; echo; }
run --rows 128 --nmma 1
run --rows 128 --nmma 1 --pdl 0
run --rows 160 --nmma 1
run --rows 256 --nmma 1
run --rows 128 --no-stream
