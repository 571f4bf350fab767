"""ctypes declarations for include/gmrf_b200.h (the C-ABI boundary).

Loads the in-tree ``_lib/libgmrf_b200.so``; there is no fallback — if the
library is missing the import of a compute entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libgmrf_b200.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class SymbolicInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("nnz_q", C.c_int64),
        ("nnz_l", C.c_int64),
        ("nnz_l_padded", C.c_int64),
        ("update_entries", C.c_int64),
        ("n_supernodes", C.c_int32),
        ("n_levels", C.c_int32),
        ("etree_height", C.c_int32),
        ("max_front", C.c_int32),
        ("flops_ref", C.c_double),
        ("flops_sn", C.c_double),
    ]


class FactorStats(C.Structure):
    _fields_ = [
        ("device_bytes", C.c_int64),
        ("launches_numeric", C.c_int64),
        ("launches_solve", C.c_int64),
        ("launches_selinv", C.c_int64),
    ]


# name -> (restype, argtypes); every symbol include/gmrf_b200.h declares.
SIGNATURES = {
    "gmrf_last_error": (C.c_char_p, []),
    "gmrf_version": (C.c_int, []),
    "gmrf_nd_order": (C.c_int, [C.c_int32, i64p, i32p, i32p]),
    "gmrf_symbolic_analyze": (C.c_int, [C.c_int32, i64p, i32p, i32p, C.POINTER(C.c_void_p)]),
    "gmrf_symbolic_info": (C.c_int, [C.c_void_p, C.POINTER(SymbolicInfo)]),
    "gmrf_symbolic_export": (C.c_int, [C.c_void_p, i32p, i32p, i64p]),
    "gmrf_symbolic_free": (None, [C.c_void_p]),
    "gmrf_factor_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "gmrf_factor_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmrf_factor_numeric": (C.c_int, [C.c_void_p, f64p, i32p]),
    "gmrf_factor_numeric_device": (C.c_int, [C.c_void_p, C.c_void_p, i32p]),
    "gmrf_solve": (C.c_int, [C.c_void_p, C.c_int, C.c_int32, f64p, f64p]),
    "gmrf_solve_device": (C.c_int, [C.c_void_p, C.c_int, C.c_int32, C.c_void_p, C.c_void_p]),
    "gmrf_selinv_diag": (C.c_int, [C.c_void_p, f64p]),
    "gmrf_selinv_diag_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmrf_selinv_pattern_nnz": (C.c_int, [C.c_void_p, i64p]),
    "gmrf_selinv_pattern": (C.c_int, [C.c_void_p, i64p, i32p, f64p]),
    "gmrf_factor_l": (C.c_int, [C.c_void_p, i64p, i32p, f64p, i32p]),
    "gmrf_factor_stats": (C.c_int, [C.c_void_p, C.POINTER(FactorStats)]),
    "gmrf_factor_free": (None, [C.c_void_p]),
    "gmrf_bench_fp64": (C.c_int, [f64p, f64p]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def ptr(a, t):
    """numpy array -> ctypes pointer (None passes NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(t)
