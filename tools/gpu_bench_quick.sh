mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(json.dumps({k: d[k] for k in ['value','e2e','roofline','cpu_baseline']}, indent=1)); print('q4', d['q4']['value'], d['q4']['h2d_frac_of_link_peak']); p=d['prefill']; print('prefill', p['value'], p['bubble_fraction'], p['expert_gemm_tflops'], p['expert_gemm_tensor_frac'])"; tail -3 gpurun_out/bench.err
