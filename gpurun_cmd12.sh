mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_kern.log 2>&1; echo "kernels rc=$?"; tail -3 gpurun_out/t_kern.log
timeout 300 python tools/op_latency_probe.py > gpurun_out/latprobe2.json 2>&1; tail -c 600 gpurun_out/latprobe2.json
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_configs_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_eng.log 2>&1; echo "engine rc=$?"; tail -3 gpurun_out/t_eng.log
timeout 600 python -u bench.py --no-prefill --no-q4 --no-ablation --no-cpu-baseline --no-x22b --sweep off --steps 2 > gpurun_out/bench_res.json 2> gpurun_out/bench_res.err; echo bench rc=$?
