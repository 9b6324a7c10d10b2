mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(json.dumps({k: d[k] for k in ['value','e2e','roofline']}, indent=1)); print('q4', d['q4']['value'], 'prefill', d['prefill']['value'], d['prefill']['bubble_fraction'])"; tail -3 gpurun_out/bench.err
