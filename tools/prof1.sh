set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_kernels.py --iters 20 --json gpurun_out/micro.json 2>&1 | tail -40
timeout 300 python tools/profile_kernels.py --iters 20 --rows 512 --only ffn 2>&1 | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 6 -c 2 -o gpurun_out/prof_ffn python tools/profile_kernels.py --only ffn --iters 2 > gpurun_out/ncu_ffn.log 2>&1
tail -5 gpurun_out/ncu_ffn.log
