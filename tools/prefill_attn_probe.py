import sys, torch
sys.path.insert(0, '.')
from paper_2502_06888_b200 import kernels as K
dev = torch.device('cuda:0')
width = (32 + 16) * 128
qkv = torch.randn(32 * 512, width, dtype=torch.bfloat16, device=dev)
out = torch.empty(32 * 512, 32 * 128, dtype=torch.bfloat16, device=dev)
import os
K.tune(K.TUNE_PREFILL_TC, int(os.environ.get("TC", "1")))
for _ in range(3):
    K.attn_prefill(qkv, 32, 512, 32, 8, 128, 260, 4, 128 ** -0.5, out)
torch.cuda.synchronize()
