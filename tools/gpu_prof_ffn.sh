# --set full of one decode-shaped expert FFN (M = 128 rows, Mixtral-8x7B expert):
# the two weight-streaming GEMM launches of kl_expert_ffn -> roofline traffic.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_stream" -s 6 -c 2 \
   -o gpurun_out/prof_ffn_r01c python tools/profile_kernels.py --only ffn --rows 128 --iters 12 > gpurun_out/ncu_ffn_r01c.log 2>&1
tail -1 gpurun_out/ncu_ffn_r01c.log
