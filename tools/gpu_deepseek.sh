mkdir -p gpurun_out
timeout 900 python tools/deepseek_run.py --bs 32 --cap 24e9 --steps 3 > gpurun_out/deepseek.json 2> gpurun_out/deepseek.err; cat gpurun_out/deepseek.json; tail -3 gpurun_out/deepseek.err
