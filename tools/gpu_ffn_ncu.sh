# ncu --set full of one expert FFN (SwiGLU GEMM + down GEMM, K-blocked
# weights, M = 128) after warm-up; summarised into profiles/ncu_expert_ffn.json
# by tools/ncu_ffn_traffic.py (run here, on the CPU box).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_stream_kernel -s 6 -c 2 \
  -o gpurun_out/r02_ffn_full -f python tools/profile_kernels.py --only ffn --iters 4 > gpurun_out/ncu_ffn.log 2>&1
tail -2 gpurun_out/ncu_ffn.log
