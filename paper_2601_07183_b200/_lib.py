"""ctypes declarations for librairs.so (include/rairs.h). Marshalling only.

The library is built in-tree (``make -C paper_2601_07183_b200/csrc``) and
loaded from this package directory. There is no fallback: if the shared
library is missing or fails to load, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librairs.so")
CSRC = os.path.join(_HERE, "csrc")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64
_F32 = ctypes.c_float

RAIRS_OK = 0
STATUS_NAMES = {0: "RAIRS_OK", -1: "RAIRS_E_INVALID", -2: "RAIRS_E_OOM", -3: "RAIRS_E_CUDA",
                -4: "RAIRS_E_UNSUPPORTED", -5: "RAIRS_E_INTERNAL"}

# every symbol include/rairs.h declares (tests check the export table)
EXPORTED_SYMBOLS = [
    "rairs_default_params", "rairs_train", "rairs_build_from_trained", "rairs_build_index",
    "rairs_index_free", "rairs_index_get_info", "rairs_search", "rairs_search_host",
    "rairs_search_debug", "rairs_merge_topk", "rairs_exact_knn", "rairs_export_trained",
    "rairs_export_assignment", "rairs_export_layout", "rairs_profile_enable",
    "rairs_profile_read", "rairs_profile_read_kernel", "rairs_last_error", "rairs_version", "rairs_set_coarse_mode",
    "rairs_certify_fallbacks", "rairs_set_scan_mode", "rairs_profile_kernels",
    "rairs_search_plan", "rairs_add", "rairs_remove_ids", "rairs_get_stats",
    "rairs_search_host_async", "rairs_set_seil_layout",
]


class BuildParams(ctypes.Structure):
    _fields_ = [("nlist", _I32), ("M", _I32), ("nbits", _I32), ("assignment", _I32),
                ("lambda_", _F32), ("n_cands", _I32), ("strict", _I32),
                ("kmeans_iters", _I32), ("train_sample", _I64), ("seed", _U64),
                ("shard_id", _I32), ("nshards", _I32)]


class IndexInfo(ctypes.Structure):
    _fields_ = [("n", _I64), ("d", _I32), ("nlist", _I32), ("M", _I32), ("M_pad", _I32),
                ("n_slots", _I64), ("n_cells", _I64), ("n_refs", _I64), ("n_double", _I64),
                ("max_refs_per_list", _I32), ("shard_id", _I32), ("nshards", _I32),
                ("device_bytes", _I64), ("n_live", _I64), ("has_ids", _I32)]


class Stats(ctypes.Structure):
    _fields_ = [("searches", _I64), ("queries", _I64), ("dco_total", _I64), ("refine_total", _I64),
                ("certify_fallbacks", _I64), ("ms_coarse", ctypes.c_double),
                ("ms_scan", ctypes.c_double), ("ms_refine", ctypes.c_double)]


class RairsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def build_library(force: bool = False) -> str:
    """Compile librairs.so for sm_100a with nvcc (cross-compiles without a GPU)."""
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cu", ".cuh", "Makefile"))]
    srcs.append(os.path.join(os.path.dirname(_HERE), "include", "rairs.h"))
    stale = (not os.path.exists(LIB_PATH) or
             max(os.path.getmtime(s) for s in srcs) > os.path.getmtime(LIB_PATH))
    if force or stale:
        subprocess.check_call(["make", "-s", "-j4", "-C", CSRC])
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librairs.so not built: run `make -C {CSRC}` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    L.rairs_last_error.restype = ctypes.c_char_p
    L.rairs_version.restype = ctypes.c_char_p
    L.rairs_default_params.argtypes = [ctypes.POINTER(BuildParams), _I32, _I32]
    L.rairs_default_params.restype = None
    PP = ctypes.POINTER(BuildParams)
    sigs = {
        "rairs_train": [_P, _I64, _I32, PP, _P, _P, _P],
        "rairs_build_from_trained": [_P, _I64, _I32, _P, _P, _P, PP, _P, ctypes.POINTER(_P)],
        "rairs_build_index": [_P, _I64, _I32, _P, PP, _P, ctypes.POINTER(_P)],
        "rairs_index_free": [_P],
        "rairs_index_get_info": [_P, ctypes.POINTER(IndexInfo)],
        "rairs_search": [_P, _P, _I64, _I32, _I32, _I32, _P, _P, _P, _P],
        "rairs_search_host": [_P, _P, _I64, _I32, _I32, _I32, _P, _P, _P],
        "rairs_search_host_async": [_P, _P, _I64, _I32, _I32, _I32, _P, _P, _P],
        "rairs_search_debug": [_P, _P, _I64, _I32, _I32, _I32] + [_P] * 10,
        "rairs_merge_topk": [_P, _P, _I32, _I64, _I32, _P, _P, _P],
        "rairs_exact_knn": [_P, _I64, _I32, _P, _I64, _I32, _P, _P, _P],
        "rairs_export_trained": [_P, _P, _P, _P],
        "rairs_export_assignment": [_P, _P, _P, _P, _P],
        "rairs_export_layout": [_P] * 9,
        "rairs_profile_enable": [_P, _I32],
        "rairs_profile_read": [_P, _P, _P, _I32],
        "rairs_profile_read_kernel": [_P, _P, _P, _I32],
        "rairs_set_coarse_mode": [_P, _I32],
        "rairs_certify_fallbacks": [_P, _P, _I32],
        "rairs_set_scan_mode": [_P, _I32],
        "rairs_set_seil_layout": [_P, _I32],
        "rairs_profile_kernels": [_P, _P, _I32],
        "rairs_search_plan": [_P, _I64, _I32, _I32, _I32, _P, _P],
        "rairs_add": [_P, _P, _I64, _P, _P, _P],
        "rairs_remove_ids": [_P, _P, _I64, _P, _P],
        "rairs_get_stats": [_P, ctypes.POINTER(Stats), _I32],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    _lib = L
    return L


def check(status: int, what: str):
    if status != RAIRS_OK:
        msg = lib().rairs_last_error()
        raise RairsError(status, f"{what}: {msg.decode() if msg else ''}")
