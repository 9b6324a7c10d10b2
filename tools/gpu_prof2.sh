mkdir -p gpurun_out
# 1) launch list of the bench command (one timed decode step after 3 warm-up steps)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 13950 -c 4600 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.out 2>&1
tail -3 gpurun_out/ncu_bench.out
# 2) full sets of the decode-shaped expert FFN GEMMs (+ split-K reduce) and the decode attention
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|splitk|attn_decode" -s 12 -c 6 \
   -o gpurun_out/prof_r01 python tools/profile_kernels.py --iters 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
# 3) reference arm (CPU port) timing
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err
cat gpurun_out/ref_arm.json; tail -3 gpurun_out/ref_arm.err
