"""Phase trace of the o-projection (residual epilogue) through the
weight-streaming GEMM (forced), M = 64. python tools/oproj_trace.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06888_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
bf = torch.bfloat16
d = 4096
for epi, nm in ((1, "residual"), (0, "store")):
    wo = torch.randn(d, d, dtype=bf, device=dev) * 0.02
    ao = torch.randn(64, d, dtype=bf, device=dev)
    h = torch.randn(64, d, dtype=bf, device=dev)
    K.tune(K.TUNE_STREAM_GEMM, 2)
    K.tune(99, 128)
    for _ in range(3):
        K.gemm(ao, wo, c=h, residual=h if epi == 1 else None, epilogue=epi)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (256 * 12))()
    K._lib.kl_stream_trace(buf, 256)
    K.gemm(ao, wo, c=h, residual=h if epi == 1 else None, epilogue=epi)
    torch.cuda.synchronize()
    K._lib.kl_stream_trace(buf, 256)
    K.tune(99, 0)
    K.tune(K.TUNE_STREAM_GEMM, 1)
    a = np.array(buf, dtype=np.float64).reshape(256, 12)[:148]
    t0 = a[:, 0][a[:, 0] > 0].min()
    rel = (a - t0) / 1e3
    rel[a == 0] = np.nan
    names = ["start", "mma0", "mma_end", "epi_last", "flags_ok", "landed", "sums_done", "end", "contrib0", "published"]
    print(nm)
    for i, n in enumerate(names):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {n:10s} med {np.nanmedian(col):7.2f}  min {np.nanmin(col):7.2f}  max {np.nanmax(col):7.2f}")
