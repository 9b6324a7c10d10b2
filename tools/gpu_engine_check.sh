# Engine GPU tests + in-step op timing + a short headline/resident bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_configs_gpu.py tests/test_ep_loopback_gpu.py -m gpu -q -x > gpurun_out/engine_tests.log 2>&1; tail -3 gpurun_out/engine_tests.log
timeout 300 python tools/op_timing.py --steps 1 > gpurun_out/op_timing.txt 2>&1; tail -12 gpurun_out/op_timing.txt
timeout 900 python bench.py --no-prefill --no-q4 --no-ablation --no-cpu-baseline --no-x22b --sweep off > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench rc=$?
