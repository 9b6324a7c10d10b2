"""The C-ABI boundary (no GPU needed): the shared library loads and exports
every entry point include/klotski/*.h declares; no-GPU calls fail loudly."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", "klotski", h) for h in ("kernels.h", "engine.h")]


def declared(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kl_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_06888_b200 import load_native
    return load_native()


@pytest.mark.parametrize("header", HEADERS, ids=os.path.basename)
def test_every_declared_symbol_is_exported(lib, header):
    names = declared(header)
    assert len(names) >= 8
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def test_abi_version_and_error_strings(lib):
    assert lib.kl_abi_version() == 1
    lib.kl_error_string.restype = C.c_char_p
    assert b"invalid" in lib.kl_error_string(-1)


def test_invalid_arguments_rejected_without_device(lib):
    # Shape validation happens before any CUDA call.
    assert lib.kl_gemm_bf16(None, 0, 0, 4, 60, None, 64, None, 64, None, 0, None) == -1
    assert lib.kl_gate_topk(None, None, None, 4, 100, 8, 2, C.c_float(1e-5), 0, None, None, None, None, None, None,
                            None) == -1


def test_engine_create_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_06888_b200.engine import DeviceError, Engine
    with pytest.raises(DeviceError, match="DeviceError"):
        Engine({"model": {"preset": "tiny"}})


def test_engine_errors_map_to_moesim_types(lib):
    """Config errors raised before any device call arrive as the moesim class
    (KL_ECONFIG / KL_EPARSE), not a generic failure."""
    import ctypes as C
    from paper_2502_06888_b200.engine import ConfigError, Engine, EngineError, ParseError
    with pytest.raises(ConfigError):
        Engine({"model": {"preset": "no-such-model"}})
    h = C.c_void_p()
    assert lib.kl_engine_create(b"{not json", C.byref(h)) == 5
    assert not h.value
    assert issubclass(ParseError, EngineError) and issubclass(ConfigError, ValueError)


def test_package_has_no_cpu_fallback(monkeypatch, tmp_path):
    import paper_2502_06888_b200 as pkg
    monkeypatch.setattr(pkg, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        pkg.load_native()
