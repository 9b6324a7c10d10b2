mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_stream -s 4 -c 2 -o gpurun_out/prof_stream python tools/profile_kernels.py --only ffn --rows 128 --iters 2 > gpurun_out/ncu_stream.log 2>&1
tail -3 gpurun_out/ncu_stream.log
