import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2502_06888_b200 import kernels as K
import oracle.pyoracle as orc
from tests.test_kernels_gpu import to_dev, to_bits
cuda = torch.device("cuda:0")
for (T, Hq, Hkv, hd, cap, p) in [(64, 32, 8, 128, 260, 600), (37, 32, 8, 128, 260, 200), (300, 8, 2, 64, 40, 39)]:
    width = (Hq + 2 * Hkv) * hd
    q = orc.normal_bf16(T * width, 61, 1.0).reshape(T, width)
    kc = orc.normal_bf16(T * cap * Hkv * hd, 62, 1.0)
    vc = orc.normal_bf16(T * cap * Hkv * hd, 63, 1.0)
    base = [p, max(p - 3, 0), p // 2, 1, p]
    pos = np.array([base[i % 5] for i in range(T)], np.int32)
    seq = np.array(list(range(T))[::-1], np.int32)
    ref = orc.bits_to_f32(orc.attn_decode(q, width, pos, seq, Hq, Hkv, hd, kc, vc, cap, hd ** -0.5)).reshape(T, Hq, hd)
    for mma in (1, 0):
        K.tune(K.TUNE_DECODE_MMA, mma)
        out = torch.empty(T, Hq * hd, dtype=torch.bfloat16, device=cuda)
        K.attn_decode_split(to_dev(q, cuda), width, torch.from_numpy(pos).to(cuda), torch.from_numpy(seq).to(cuda),
                            Hq, Hkv, hd, to_dev(kc, cuda), to_dev(vc, cuda), cap, 4, hd ** -0.5, out)
        torch.cuda.synchronize()
        got = orc.bits_to_f32(to_bits(out)).reshape(T, Hq, hd)
        err = np.abs(got - ref).max(axis=2)  # T x Hq
        bad = np.argwhere(~(err < 0.05))
        print(T, Hq, Hkv, hd, cap, "mma", mma, "bad (t,h) count", len(bad), "tokens", sorted(set(bad[:, 0].tolist()))[:20], "heads", sorted(set(bad[:, 1].tolist()))[:40])
