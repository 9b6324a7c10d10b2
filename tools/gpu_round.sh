# One GPU call: full gpu test suite (kernels first), short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -c 3000 gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err
