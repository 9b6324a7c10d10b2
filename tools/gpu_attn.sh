mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k attention 2>&1 | tail -2
timeout 300 python tools/profile_kernels.py --iters 20 --only attn --gap-ms 0.05 2>&1 | grep -A2 'attn' | grep -E 'attn|us|GBs'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_decode_split|attn_merge" -s 4 -c 2 -o gpurun_out/prof_attn python tools/profile_kernels.py --only attn --iters 2 > gpurun_out/ncu_attn.log 2>&1
