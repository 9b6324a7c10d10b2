mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_route.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_route.log
timeout 300 python tools/profile_kernels.py --only route --iters 20 --json gpurun_out/route.json > /dev/null 2>gpurun_out/route.err; cat gpurun_out/route.json | tr -d '\n '; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"combine|permute|rmsnorm" -c 12 -o gpurun_out/prof_r02_route2 -f python tools/profile_kernels.py --only route --iters 1 > gpurun_out/ncu_route2.log 2>&1; echo ncu rc=$?
timeout 600 python -u bench.py --no-prefill --no-q4 --no-ablation --no-cpu-baseline --no-x22b --sweep off --steps 2 > gpurun_out/bench_res.json 2> gpurun_out/bench_res.err; echo bench rc=$?
