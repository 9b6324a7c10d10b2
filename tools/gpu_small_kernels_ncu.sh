# ncu --set full of the decode-path small kernels (router, RMSNorm, permute,
# combine, RoPE/KV append) at decode and prefill sizes, one launch each after
# warm-up (tools/profile_kernels.py --only route / attn).
mkdir -p gpurun_out
for k in gate_topk_block rmsnorm_row permute_rank permute_scatter combine_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/r02_full_$k -f python tools/profile_kernels.py --only route > gpurun_out/ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:rope_append -s 3 -c 1 \
  -o gpurun_out/r02_full_rope -f python tools/profile_kernels.py --only attn > gpurun_out/ncu_rope.log 2>&1
