"""ctypes loader for the in-tree libbolt.so (C ABI of include/bolt.h).

There is no fallback: if the shared library is missing or fails to load, the
import of the compute functions raises.  Build it with
``python -m paper_1706_10283_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# BOLT_LIB selects another in-tree build (tools/ use libbolt_prof.so)
LIB_PATH = os.path.join(_PKG, os.environ.get("BOLT_LIB", "libbolt.so"))

BOLT_OK = 0
STATUS = {0: "BOLT_OK", 1: "BOLT_E_NULL", 2: "BOLT_E_SHAPE", 3: "BOLT_E_RANGE", 4: "BOLT_E_ALIGN",
          5: "BOLT_E_DEVICE", 6: "BOLT_E_CUDA", 7: "BOLT_E_WORKSPACE"}

# every symbol include/bolt.h declares, with (argtypes, restype)
_P, _I64, _I32, _F32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
SIGNATURES = {
    "bolt_version": ([], ctypes.c_char_p),
    "bolt_last_error": ([], ctypes.c_char_p),
    "bolt_codes_words": ([_I64, _I32], _I64),
    "bolt_encode": ([_P, _I64, _I32, _I64, _P, _I32, _P, _P], _I32),
    "bolt_encode_ex": ([_P, _I64, _I32, _I64, _P, _I32, _P, _I32, _P], _I32),
    "bolt_encode_append": ([_P, _I64, _I32, _I64, _P, _I32, _P, _I64, _P], _I32),
    "bolt_pack_codes": ([_P, _I64, _I32, _P, _P], _I32),
    "bolt_unpack_codes": ([_P, _I64, _I32, _P, _P], _I32),
    "bolt_build_luts": ([_P, _I64, _I32, _I64, _P, _I32, _I32, _P, _P], _I32),
    "bolt_build_luts_f64": ([_P, _I64, _I32, _I64, _P, _I32, _I32, _P, _P], _I32),
    "bolt_quantize_luts": ([_P, _I64, _I32, _F32, _P, _P, _P], _I32),
    "bolt_build_quantized_luts": ([_P, _I64, _I32, _I64, _P, _I32, _I32, _F32, _P, _P, _P, _P], _I32),
    "bolt_scan": ([_P, _I64, _I32, _P, _I64, _P, _I64, _P], _I32),
    "bolt_scan_dequant": ([_P, _I64, _I32, _P, _I64, _F32, _F32, _P, _I64, _P], _I32),
    "bolt_scan_ex": ([_P, _I64, _I32, _P, _I64, _P, _I64, _I32, _P], _I32),
    "bolt_scan_dequant_ex": ([_P, _I64, _I32, _P, _I64, _F32, _F32, _P, _I64, _I32, _P], _I32),
    "bolt_topk_workspace_bytes": ([_I64, _I32, _I64, _I32], _SZ),
    "bolt_topk": ([_P, _I64, _I32, _P, _I64, _I32, _I32, _I64, _P, _P, _SZ, _P], _I32),
    "bolt_topk_plan": ([_I64, _I32, _I64, _I32, _I32, _P, _P], _I32),
    "bolt_topk_workspace_bytes_ex": ([_I64, _I32, _I64, _I32, _I32], _SZ),
    "bolt_topk_ex": ([_P, _I64, _I32, _P, _I64, _I32, _I32, _I64, _P, _P, _SZ, _I32, _P], _I32),
    "bolt_topk_merge": ([_P, _I32, _I64, _I32, _P, _P], _I32),
    "bolt_keys_split": ([_P, _I64, _I32, _P, _P, _P], _I32),
    "bolt_scan_f32": ([_P, _I64, _I32, _P, _I64, _P, _I64, _P], _I32),
    "bolt_topk_f32_workspace_bytes": ([_I64, _I32, _I64, _I32], ctypes.c_size_t),
    "bolt_topk_f32": ([_P, _I64, _I32, _P, _I64, _I32, _I32, _I64, _P, _P, ctypes.c_size_t, _P], _I32),
    "bolt_keys_split_f32": ([_P, _I64, _I32, _P, _P, _P], _I32),
    "bolt_search_host_workspace_bytes": ([_I64, _I32, _I32, _I64, _I32], _SZ),
    "bolt_search_host": ([_P, _I64, _I32, _P, _I64, _P, _I32, _I32, _F32, _P, _I32, _P, _P, _SZ, _P], _I32),
    "bolt_search_host_ex": ([_P, _I64, _I32, _P, _I64, _P, _I32, _I32, _F32, _P, _I32, _I64, _P, _P, _SZ, _P], _I32),
    "bolt_search_host_pipelined_ex": ([_P, _I64, _I32, _P, _I64, _P, _I32, _I32, _F32, _P, _I32, _I64, _P, _P, _SZ,
                                       _I32, _P, _P], _I32),
    "bolt_search_host_pipelined_workspace_bytes": ([_I64, _I32, _I32, _I64, _I32, _I32], _SZ),
    "bolt_search_host_pipelined": ([_P, _I64, _I32, _P, _I64, _P, _I32, _I32, _F32, _P, _I32, _P, _P, _SZ, _I32,
                                    _P, _P], _I32),
    "bolt_kmeans_workspace_bytes": ([_I64, _I32, _I32], _SZ),
    "bolt_kmeans": ([_P, _I64, _I32, _I64, _I32, _P, _I32, _P, _P, _SZ, _P], _I32),
    "bolt_calibrate_workspace_bytes": ([_I64, _I32], _SZ),
    "bolt_calibrate": ([_P, _I64, _I32, _P, _P, _P, _P, _SZ, _P], _I32),
    "bolt_debug_counters": ([_P, _I32], _I32),
}


class BoltError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_1706_10283_b200.build` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            if not hasattr(lib, name) and (name.startswith("bolt_debug_") or os.environ.get("BOLT_LIB")):
                continue  # absent from an older build loaded for a tools/ A/B run
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def call(name: str, *args) -> None:
    st = getattr(load(), name)(*args)
    if st != BOLT_OK:
        raise BoltError(name, st, load().bolt_last_error().decode())
