# Tensor-pipe evidence for the prefill expert GEMMs (M = 8192 rows of one expert).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_tcgen05|attn_prefill_tc" -s 2 -c 3 \
   -o gpurun_out/prof_prefill python tools/profile_kernels.py --only ffn --rows 8192 --iters 1 > gpurun_out/ncu_prefill.log 2>&1
tail -2 gpurun_out/ncu_prefill.log
cat > /tmp/pfattn.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2502_06888_b200 import kernels as K
dev = torch.device('cuda:0')
width = (32 + 16) * 128
qkv = torch.randn(16 * 512, width, dtype=torch.bfloat16, device=dev)
out = torch.empty(16 * 512, 32 * 128, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    K.attn_prefill(qkv, 16, 512, 32, 8, 128, 260, 4, 128 ** -0.5, out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_prefill_tc" -s 1 -c 1 \
   -o gpurun_out/prof_prefill_attn python /tmp/pfattn.py > gpurun_out/ncu_prefill_attn.log 2>&1
tail -2 gpurun_out/ncu_prefill_attn.log
