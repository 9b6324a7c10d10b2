# Round-1 (session 2) profiles: launch list of one bench decode step and
# --set full captures of the decode FFN (bf16 + Q4T), split-KV decode
# attention and the tcgen05 prefill attention.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv \
   --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-q4 --no-prefill \
   > gpurun_out/ncu_bench.out 2>&1
tail -2 gpurun_out/ncu_bench.out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_stream|attn_decode_split|attn_merge" -s 20 -c 6 \
   -o gpurun_out/prof_r01b_decode python tools/profile_kernels.py --iters 2 > gpurun_out/ncu_full1.log 2>&1
tail -2 gpurun_out/ncu_full1.log
cat > /tmp/q4prof.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2502_06888_b200 import kernels as K
d, f, M = 4096, 14336, 128
dev = torch.device('cuda:0')
w = (torch.randn(3 * d * f, dtype=torch.bfloat16, device=dev) * 0.02)
q13 = K.quantize_q4(w[: 2 * f * d].view(2 * f, d)); q2 = K.quantize_q4(w[2 * f * d:].view(d, f))
x = torch.randn(1024, d, dtype=torch.bfloat16, device=dev)
y = torch.empty_like(x); h = torch.empty(M, f, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    K.expert_ffn_q4(x, 0, M, q13, q2, d, f, y, h)
torch.cuda.synchronize()
# prefill attention: 8 seqs x 512, Mixtral heads
width = (32 + 16) * 128
qkv = torch.randn(8 * 512, width, dtype=torch.bfloat16, device=dev)
out = torch.empty(8 * 512, 32 * 128, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    K.attn_prefill(qkv, 8, 512, 32, 8, 128, 260, 4, 128 ** -0.5, out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_stream|attn_prefill_tc" -s 2 -c 4 \
   -o gpurun_out/prof_r01b_q4_prefill python /tmp/q4prof.py > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full2.log
