"""moesim — the reference's Python package name (proj/python/moesim,
proj/CMakeLists.txt:28-37), backed by this repo's build: `moesim._core` is the
pybind11 module paper_2502_06888_b200/_core (planner, schedule, simulator,
trace API of include/moesim/*.hpp)."""
import sys

from paper_2502_06888_b200 import load_native as _load_native

_load_native()
from paper_2502_06888_b200 import _core  # noqa: E402

sys.modules[__name__ + "._core"] = _core
from paper_2502_06888_b200._core import *  # noqa: E402,F401,F403
