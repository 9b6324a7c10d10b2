"""B200-native Klotski layer-execution path (arXiv 2502.06888).

Native pieces (built in-tree by `make` / `__graft_entry__.build()`):
  libklotski.so  - moesim C++ API (include/moesim) + B200 engine + sm_100a kernels
                   behind the C-ABI in include/klotski/*.h
  _core*.so      - pybind11 module mirroring the reference's `moesim._core`

There is no CPU fallback: importing the kernel or engine wrappers raises if the
native library is missing.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libklotski.so")


def load_native():
    """Load libklotski.so (RTLD_GLOBAL so _core and libparity resolve against it)."""
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built; run `make` (or __graft_entry__.build()) first. "
            "There is no CPU fallback for the B200 path.")
    return ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
