"""ctypes access to the parity driver (oracle/parity_driver.cpp) compiled
twice: against the reference library (oracle/_ref/libref_parity.so, the
oracle) and against this repo's moesim implementation (libparity.so).
Test infrastructure only."""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libref_parity.so")
MINE_LIB = os.path.join(ROOT, "paper_2502_06888_b200", "libparity.so")


class Driver:
    def __init__(self, path):
        if "paper_2502_06888_b200" in path:
            from paper_2502_06888_b200 import load_native
            load_native()
        self.lib = C.CDLL(path)
        self.lib.parity_request.argtypes = [C.c_char_p]
        self.lib.parity_request.restype = C.c_void_p
        self.lib.parity_free.argtypes = [C.c_void_p]

    def __call__(self, req):
        p = self.lib.parity_request(json.dumps(req).encode())
        try:
            return json.loads(C.string_at(p).decode())
        finally:
            self.lib.parity_free(p)


_cache = {}


def ref():
    if "ref" not in _cache:
        _cache["ref"] = Driver(REF_LIB)
    return _cache["ref"]


def mine():
    if "mine" not in _cache:
        _cache["mine"] = Driver(MINE_LIB)
    return _cache["mine"]


def request_for_engine(info, cfg):
    """Reference request reproducing an engine's plan + replay schedule."""
    spec, prof = info["spec"], info["profile"]
    w = cfg["workload"]
    req = {
        "model": {"preset": "toy", "n_layers": spec["n_layers"], "n_experts": spec["n_experts"],
                  "top_k": spec["top_k"], "expert_bytes": spec["expert_bytes"],
                  "attention_bytes": spec["attention_bytes"], "gate_bytes": spec["gate_bytes"],
                  "kv_bytes_per_token": spec["kv_bytes_per_token"]},
        "hw": dict(prof),
        "workload": {"batch_size": w["batch_size"], "n_batches": info["n_batches"], "prompt_len": w["prompt_len"],
                     "gen_len": w["gen_len"]},
        "skew": cfg.get("skew", {"kind": "zipf", "s": 1.5}),
        "seed": cfg.get("trace_seed", 1),
        "n": info["n_batches"],
        "variant": cfg.get("variant", "klotski"),
        "working_set_override": info["working_set_bytes"],
        "streaming_kv": info["streaming_kv"],
        "sink_tokens": info["sink_tokens"],
        "window_tokens": info["window_tokens"],
        "simulate": False,
    }
    if cfg.get("quant"):
        req["quant"] = True
    return req
