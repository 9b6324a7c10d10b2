# PDL-window L2 prefetch of weight units (KL_TUNE_STREAM_PRE_L2): attention
# op parts and the expert FFN at 0 / 8 / 16 / 32 units.
mkdir -p gpurun_out/pl2
for U in 0 8 16 32; do
  timeout 300 python tools/profile_kernels.py --only attnop --pre-l2 $U --json gpurun_out/pl2/attn_$U.json > /dev/null 2>&1
  timeout 300 python tools/profile_kernels.py --only ffn --pre-l2 $U --json gpurun_out/pl2/ffn_$U.json > /dev/null 2>&1
  python - <<PY
import json
a=json.load(open('gpurun_out/pl2/attn_$U.json')); f=json.load(open('gpurun_out/pl2/ffn_$U.json'))
print('pre_l2=$U', 'attn_deferred', round(a['attn_op_b64_deferred_qkv']['us'],1), 'qkv_def', round(a['attn_op_part_qkv_deferred']['us'],1),
      'ffn_def', round(f['expert_ffn_deferred_graph']['us'],1), 'swiglu', round(f['gemm_swiglu_graph']['us'],1))
PY
done
