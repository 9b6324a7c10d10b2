"""4-bit expert format pinned against the REFERENCE library
(oracle/_ref, the unmodified proj/src compiled here, through the parity
driver; no GPU): the oracle's min-max fit equals moesim::fit_minmax
(quant.cpp) group by group, and the oracle's Q4T tiles dequantise to exactly
what moesim::dequantize returns for the same codes / scales / zeros in the
reference's flat QuantizedTensor order (quant.cpp:197-252). The same checks
run against this repo's moesim._core so both sides agree."""
import numpy as np
import pytest

from oracle import pyoracle as orc
from tests import parity


@pytest.fixture(scope="module")
def core():
    import moesim._core as c
    return c


def _groups():
    rows, K = 128, 256
    w = orc.normal_bf16(rows * K, 71, 0.02).reshape(rows, K)
    g = orc.bits_to_f32(w).reshape(-1, 64)
    g[3] = 0.5  # constant group (lo == hi branch)
    g[7, :] = np.linspace(-0.1, 0.3, 64, dtype=np.float32)
    return g


def _flat_from_tiles(q, rows, K):
    """Re-assemble the reference's flat group order (codes little-endian,
    one f16 scale / zero per 64-group) from Q4T tiles."""
    KB = K // 64
    packed = np.empty((rows, KB, 32), np.uint8)
    sc = np.empty((rows, KB), np.uint16)
    zr = np.empty((rows, KB), np.uint16)
    for rt in range(rows // 128):
        for kb in range(KB):
            base = (rt * KB + kb) * orc.Q4_CHUNK
            packed[rt * 128:rt * 128 + 128, kb] = q[base:base + 4096].reshape(128, 32)
            sc[rt * 128:rt * 128 + 128, kb] = np.ascontiguousarray(q[base + 4096:base + 4352]).view(np.uint16)
            zr[rt * 128:rt * 128 + 128, kb] = np.ascontiguousarray(q[base + 4352:base + 4608]).view(np.uint16)
    return packed.reshape(-1), sc.reshape(-1), zr.reshape(-1)


def test_q4_fit_matches_reference_library():
    g = _groups()
    scale, zero = orc.q4_fit_minmax(g)
    ref = parity.ref()({"quant_ops": {"fit": g.tolist(), "bits": 4}})["fit"]
    assert len(ref) == g.shape[0]
    for i, (s_ref, z_ref) in enumerate(ref):
        assert np.float32(scale[i]) == np.float32(s_ref) and np.float32(zero[i]) == np.float32(z_ref), i


def test_q4_fit_matches_repo_core(core):
    g = _groups()
    scale, zero = orc.q4_fit_minmax(g)
    for i in range(g.shape[0]):
        s_ref, z_ref = core.fit_minmax(g[i], 4)
        assert np.float32(scale[i]) == np.float32(s_ref) and np.float32(zero[i]) == np.float32(z_ref), i


def test_q4_tiles_equal_reference_library_dequantize():
    rows, K = 256, 192
    w = orc.normal_bf16(rows * K, 72, 0.05).reshape(rows, K)
    q = orc.q4_quantize_tiled(w)
    assert q.size == parity.ref()({"quant_ops": {"bytes": rows * K}})["bytes"]  # 0.28125 x bf16 bytes
    deq = orc.q4_dequantize_tiled(q, rows, K)
    packed, sc, zr = _flat_from_tiles(q, rows, K)
    ref = parity.ref()({"quant_ops": {"dequant": {"n": rows * K, "packed": packed.tolist(), "scales": sc.tolist(),
                                                  "zeros": zr.tolist()}}})["dequant"]
    ref = np.asarray(ref, np.float64).astype(np.float32)
    assert np.array_equal(ref.view(np.uint32), deq.reshape(-1).view(np.uint32))
    # Reconstruction stays within half a quantisation step per group.
    g = orc.bits_to_f32(w).reshape(-1, 64)
    s = np.repeat(sc.view(np.float16).astype(np.float32), 64)
    assert np.all(np.abs(deq.reshape(-1) - g.reshape(-1)) <= 0.5 * s + 1e-6)


def test_q4_tiles_equal_repo_core_dequantize(core):
    rows, K = 256, 192
    w = orc.normal_bf16(rows * K, 72, 0.05).reshape(rows, K)
    q = orc.q4_quantize_tiled(w)
    assert q.size == core.quantized_bytes(rows * K, core.QuantConfig())
    deq = orc.q4_dequantize_tiled(q, rows, K)
    packed, sc, zr = _flat_from_tiles(q, rows, K)
    ref = core.dequantize(packed, sc, zr, rows * K, 4, 64)
    assert np.array_equal(ref.view(np.uint32), deq.reshape(-1).view(np.uint32))
