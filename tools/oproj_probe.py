import sys, torch
sys.path.insert(0, '.')
from paper_2502_06888_b200 import kernels as K
sys.path.insert(0, 'tools')
from profile_kernels import timed_graph
dev = torch.device('cuda:0'); bf = torch.bfloat16
d, Hq, hd, Hkv = 4096, 32, 128, 8
res = {}
for M in (64, 128):
    wo = [torch.randn(d, Hq * hd, dtype=bf, device=dev) * 0.02 for _ in range(8)]
    wqkv = [torch.randn((Hq + 2 * Hkv) * hd, d, dtype=bf, device=dev) * 0.02 for _ in range(8)]
    ao = torch.randn(M, Hq * hd, dtype=bf, device=dev)
    x = torch.randn(M, d, dtype=bf, device=dev)
    h = torch.randn(M, d, dtype=bf, device=dev)
    qkv = torch.empty(M, (Hq + 2 * Hkv) * hd, dtype=bf, device=dev)
    for mode in (0, 1, 2):
        K.tune(K.TUNE_STREAM_GEMM, mode)
        t1 = timed_graph(lambda i: K.gemm(ao, wo[i % 8], c=h, residual=h, epilogue=1), 16)
        t2 = timed_graph(lambda i: K.gemm(x, wqkv[i % 8], c=qkv), 16)
        res[f"M{M}_stream{mode}"] = (round(t1 * 1e6, 1), round(t2 * 1e6, 1))
    K.tune(K.TUNE_STREAM_GEMM, 1)
print(res)
