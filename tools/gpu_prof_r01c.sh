# Round-1 (session 3) profiles: launch list of one bench decode step and a
# --set full capture of the tensor-core decode attention + the decode FFN.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv \
   --log-file gpurun_out/launches_r01d.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-q4 --no-prefill \
   > gpurun_out/ncu_bench_d.out 2>&1
tail -2 gpurun_out/ncu_bench_d.out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_stream|attn_decode_mma" -s 12 -c 4 \
   -o gpurun_out/prof_r01d_decode python tools/profile_kernels.py --iters 2 > gpurun_out/ncu_full_d.log 2>&1
tail -2 gpurun_out/ncu_full_d.log
