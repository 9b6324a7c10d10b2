"""Host-side cost per call of the C-ABI entry points on the decode path
(async enqueue only; the GPU is kept busy by a long spin so queues never
drain). python tools/host_launch_probe.py"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    d, f, Hq, Hkv, hd, bs, cap = 4096, 14336, 32, 8, 128, 64, 260
    width = (Hq + 2 * Hkv) * hd
    x = torch.randn(bs, d, dtype=bf, device=dev)
    wqkv = torch.randn(width, d, dtype=bf, device=dev)
    qkv = torch.empty(bs, width, dtype=bf, device=dev)
    w13 = torch.randn(2 * f, d, dtype=bf, device=dev)
    w2 = torch.randn(d, f, dtype=bf, device=dev)
    xp = torch.randn(128, d, dtype=bf, device=dev)
    y = torch.empty_like(xp)
    h = torch.empty(128, f, dtype=bf, device=dev)
    kc = torch.randn(bs * cap * Hkv * hd, dtype=bf, device=dev)
    vc = torch.randn_like(kc)
    pos = torch.full((bs,), 600, dtype=torch.int32, device=dev)
    seq = torch.arange(bs, dtype=torch.int32, device=dev)
    out = torch.empty(bs, Hq * hd, dtype=bf, device=dev)
    nw = torch.ones(d, dtype=bf, device=dev)
    wg = torch.randn(8, d, dtype=bf, device=dev)
    calls = {
        "gemm_qkv": lambda: K.gemm(x, wqkv, c=qkv),
        "expert_ffn": lambda: K.expert_ffn(xp, 0, 128, w13, w2, y, h),
        "attn_decode": lambda: K.attn_decode_split(qkv, width, pos, seq, Hq, Hkv, hd, kc, vc, cap, 4, hd ** -0.5, out),
        "rmsnorm": lambda: K.rmsnorm(x, nw),
        "gate_topk": lambda: K.gate_topk(x, nw, wg, 2),
    }
    flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    res = {}
    for name, fn in calls.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        flag[0] = 0
        K._lib.kl_debug_spin_flag(ctypes.c_void_p(flag.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        flag[0] = 1
        torch.cuda.synchronize()
        res[name] = round((t1 - t0) / n * 1e6, 1)
    print("host us per call (python wrapper + C-ABI enqueue):", res)


if __name__ == "__main__":
    main()
