"""ctypes bindings for include/klotski/engine.h (the B200 execution engine).

    eng = Engine({"model": {"preset": "tiny"}, "workload": {...}, "hbm_cap_bytes": ...})
    next_ids, ms = eng.step(0, prompt_ids)          # prefill
    next_ids, ms = eng.step(1)                      # decode (feeds previous tokens)
    eng.report("metrics")                           # measured RunMetrics (+ H2D stats)

No CPU fallback: construction fails if libklotski.so is missing or the GPU is
not an sm_100 part.
"""
import ctypes as C
import json

import numpy as np

from . import load_native

_lib = load_native()
_lib.kl_engine_create.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
_lib.kl_engine_create.restype = C.c_int
_lib.kl_engine_destroy.argtypes = [C.c_void_p]
_lib.kl_engine_destroy.restype = None
_lib.kl_engine_last_error.argtypes = [C.c_void_p]
_lib.kl_engine_last_error.restype = C.c_char_p
_lib.kl_engine_free_string.argtypes = [C.c_void_p]
_lib.kl_engine_free_string.restype = None
_lib.kl_engine_describe.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
_lib.kl_engine_fill_kv_synthetic.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
_lib.kl_engine_step.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
_lib.kl_engine_report.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]
_lib.kl_engine_reset_log.argtypes = [C.c_void_p]
_lib.kl_engine_read_hidden.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]


_lib.kl_measure_profile.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
_lib.kl_measure_profile.restype = C.c_int
_lib.kl_ep_unique_id.argtypes = [C.c_char_p]
_lib.kl_ep_unique_id.restype = C.c_int


def ep_unique_id():
    """NCCL unique id (hex) for an expert-parallel group; create on rank 0 and share."""
    buf = C.create_string_buffer(257)
    if _lib.kl_ep_unique_id(buf) != 0:
        raise RuntimeError("kl_ep_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.value.decode()


class EngineError(RuntimeError):
    """Base of every engine failure; subclasses mirror the moesim exception
    taxonomy (reference error.hpp:11-49) by the C-ABI return code (KL_E*)."""


class ConfigError(EngineError, ValueError):
    pass


class ValidationError(EngineError, ValueError):
    pass


class ParseError(EngineError, ValueError):
    pass


class RangeError(EngineError, IndexError):
    pass


class AccountingError(EngineError):
    pass


class DeviceError(EngineError):
    """CUDA / NCCL / OS failure under the engine (fatal for the handle)."""


class MemoryInfeasible(EngineError):
    pass


_ERRORS = {2: MemoryInfeasible, 3: ConfigError, 4: ValidationError, 5: ParseError, 6: RangeError,
           7: AccountingError, 8: DeviceError}


def _raise(rc, msg):
    raise _ERRORS.get(rc, EngineError)(msg)


def measure_profile(config, phase="decode"):
    """Planner stage 1: this GPU's per-token attention / gate / expert rates
    and pinned H2D bandwidth on the config's model shapes (kl_measure_profile)."""
    out = C.c_void_p()
    rc = _lib.kl_measure_profile(json.dumps(config).encode(), phase.encode(), C.byref(out))
    if rc != 0:
        _raise(rc, _lib.kl_engine_last_error(None).decode())
    try:
        return json.loads(C.string_at(out).decode())
    finally:
        _lib.kl_engine_free_string(out)


class Engine:
    def __init__(self, config):
        self._h = C.c_void_p()
        text = json.dumps(config).encode()
        rc = _lib.kl_engine_create(text, C.byref(self._h))
        if rc != 0:
            _raise(rc, _lib.kl_engine_last_error(None).decode())
        self.info = self._json(_lib.kl_engine_describe)
        self.n_batches = self.info["n_batches"]
        self.batch_size = self.info["batch_size"]
        self.n_seqs = self.n_batches * self.batch_size

    def _check(self, rc):
        if rc != 0:
            _raise(rc, _lib.kl_engine_last_error(self._h).decode())

    def _json(self, fn, *args):
        out = C.c_void_p()
        self._check(fn(self._h, *args, C.byref(out)))
        try:
            return json.loads(C.string_at(out).decode())
        finally:
            _lib.kl_engine_free_string(out)

    def close(self):
        if self._h:
            _lib.kl_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fill_kv_synthetic(self, positions, seed=11):
        self._check(_lib.kl_engine_fill_kv_synthetic(self._h, positions, seed))

    def step(self, step, tokens=None, want_next=True):
        """Run one step; tokens (host int32) or None to feed back the last greedy tokens."""
        tin = None
        if tokens is not None:
            tokens = np.ascontiguousarray(tokens, dtype=np.int32).reshape(-1)
            want = self.n_seqs * (self.info["prompt_len"] if step == 0 else 1)
            if tokens.size != want:
                raise EngineError(f"step {step}: expected {want} token ids, got {tokens.size}")
            tin = tokens.ctypes.data_as(C.c_void_p)
        nxt = np.empty(self.n_seqs, np.int32) if want_next else None
        ms = C.c_double()
        self._check(_lib.kl_engine_step(self._h, step, tin, nxt.ctypes.data_as(C.c_void_p) if want_next else None,
                                        C.byref(ms)))
        return nxt, ms.value

    def report(self, what="metrics"):
        return self._json(_lib.kl_engine_report, what.encode())

    def reset_log(self):
        self._check(_lib.kl_engine_reset_log(self._h))

    def read_hidden(self, n):
        out = np.empty(n, np.uint16)
        self._check(_lib.kl_engine_read_hidden(self._h, out.ctypes.data_as(C.c_void_p), n))
        return out
