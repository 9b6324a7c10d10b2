mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/deepseek_run.py --bs 32 --cap 24e9 --steps 3 > gpurun_out/deepseek.json 2> gpurun_out/deepseek.err; cat gpurun_out/deepseek.json | cut -c1-400
