mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(json.dumps({k: d[k] for k in ['value','e2e','roofline','cpu_baseline','q4','prefill']}, indent=1))"; tail -3 gpurun_out/bench.err
