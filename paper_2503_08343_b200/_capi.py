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


class SpaceTimeConfig(C.Structure):
    _fields_ = [
        ("n_el", C.c_int32), ("xa", C.c_double), ("xb", C.c_double), ("n_t", C.c_int32),
        ("t_end", C.c_double), ("diffusion", C.c_double), ("advection", C.c_double),
        ("noise_kappa", C.c_double), ("noise_alpha", C.c_int32), ("noise_tau", C.c_double),
        ("init_kappa", C.c_double), ("init_alpha", C.c_int32), ("init_tau", C.c_double),
        ("tau", C.c_double), ("eps", C.c_double), ("dirichlet", C.c_int32),
        ("ic_noise_prec", C.c_double), ("residual", C.c_int32), ("pde_noise_prec", C.c_double),
        ("gn_max_iters", C.c_int32), ("gn_decrement_tol", C.c_double), ("gn_armijo_c", C.c_double),
        ("gn_shrink", C.c_double), ("gn_max_backtracks", C.c_int32), ("dim", C.c_int32),
    ]


class GnIter(C.Structure):
    _fields_ = [("iter", C.c_int32), ("objective", C.c_double), ("decrement", C.c_double),
                ("step_size", C.c_double), ("backtracks", C.c_int32)]


class SpaceTimeInfo(C.Structure):
    _fields_ = [
        ("setup_host_ms", C.c_double), ("init_ms", C.c_double), ("assemble_ms", C.c_double),
        ("condition_ms", C.c_double),
        ("gn_ms", C.c_double), ("laplace_ms", C.c_double), ("selinv_ms", C.c_double),
        ("numeric_ms", C.c_double), ("n_factorizations", C.c_int32),
        ("kernel_launches", C.c_int64), ("n", C.c_int32), ("n_space", C.c_int32),
        ("n_res", C.c_int32), ("nnz_pattern", C.c_int64), ("nnz_l", C.c_int64),
        ("nnz_l_padded", C.c_int64), ("flops_ref", C.c_double), ("flops_sn", C.c_double),
        ("factor_device_bytes", C.c_int64),
        ("numeric_pure_ms", C.c_double), ("n_pure_factorizations", C.c_int32),
    ]


vp = C.c_void_p


class MaternConfig(C.Structure):
    """gmrf_matern_config_t: P1 mesh + MaternSpec."""
    _fields_ = [("dim", C.c_int32), ("n_el", C.c_int32), ("xa", C.c_double), ("xb", C.c_double),
                ("kappa", C.c_double), ("alpha", C.c_int32), ("tau", C.c_double)]


class RegressionInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("nnz_pattern", C.c_int64),
                ("nnz_l", C.c_int64), ("setup_host_ms", C.c_double), ("run_ms", C.c_double),
                ("flops_ref", C.c_double), ("kernel_launches", C.c_int64)]


class CgConfig(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_iter", C.c_int64),
                ("preconditioner", C.c_int32)]


class CgResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("final_residual", C.c_double),
                ("converged", C.c_int32)]


class Msg(C.Structure):
    """gmrf_msg_t: one message of an exchange point of a partitioned factor."""
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("tag", C.c_int32),
                ("phase", C.c_int32), ("dptr", C.c_void_p), ("count", C.c_int64)]


# int (*gmrf_exchange_fn)(void* ctx, const gmrf_msg_t* msgs, int32_t count, void* cuda_stream)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(Msg), C.c_int32, C.c_void_p)

# name -> (restype, argtypes); every symbol include/gmrf_b200.h declares.
SIGNATURES = {
    "gmrf_last_error": (C.c_char_p, []),
    "gmrf_version": (C.c_int, []),
    "gmrf_nd_order": (C.c_int, [C.c_int32, i64p, i32p, i32p]),
    "gmrf_symbolic_analyze": (C.c_int, [C.c_int32, i64p, i32p, i32p, C.POINTER(C.c_void_p)]),
    "gmrf_symbolic_info": (C.c_int, [C.c_void_p, C.POINTER(SymbolicInfo)]),
    "gmrf_symbolic_export": (C.c_int, [C.c_void_p, i32p, i32p, i64p]),
    "gmrf_symbolic_free": (None, [C.c_void_p]),
    "gmrf_symbolic_supernodes": (C.c_int, [C.c_void_p, i32p, i32p, i32p, i32p]),
    "gmrf_factor_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "gmrf_factor_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmrf_factor_numeric": (C.c_int, [C.c_void_p, f64p, i32p]),
    "gmrf_factor_numeric_device": (C.c_int, [C.c_void_p, C.c_void_p, i32p]),
    "gmrf_solve": (C.c_int, [C.c_void_p, C.c_int, C.c_int32, f64p, f64p]),
    "gmrf_solve_device": (C.c_int, [C.c_void_p, C.c_int, C.c_int32, C.c_void_p, C.c_void_p]),
    "gmrf_selinv_diag": (C.c_int, [C.c_void_p, f64p]),
    "gmrf_selinv_diag_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmrf_sample_direct": (C.c_int, [C.c_void_p, f64p, C.c_int32, C.c_uint64, f64p]),
    "gmrf_rbmc_variance": (C.c_int, [C.c_void_p, f64p, f64p, C.c_int32, C.c_uint64, f64p]),
    "gmrf_selinv_pattern_nnz": (C.c_int, [C.c_void_p, i64p]),
    "gmrf_selinv_pattern": (C.c_int, [C.c_void_p, i64p, i32p, f64p]),
    "gmrf_factor_l": (C.c_int, [C.c_void_p, i64p, i32p, f64p, i32p]),
    "gmrf_factor_stats": (C.c_int, [C.c_void_p, C.POINTER(FactorStats)]),
    "gmrf_factor_free": (None, [C.c_void_p]),
    "gmrf_bench_fp64": (C.c_int, [f64p, f64p]),
    "gmrf_rng_fill": (C.c_int, [C.c_uint64, C.c_int32, C.c_int64, f64p]),
    "gmrf_rng_draw": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, f64p]),
    "gmrf_cg_solve": (C.c_int, [C.c_int32, i64p, i32p, f64p, f64p, f64p, C.POINTER(CgConfig),
                                f64p, C.POINTER(CgResult)]),
    "gmrf_sample_cg": (C.c_int, [C.c_int32, i64p, i32p, f64p, C.c_int32, i64p, i32p, f64p, f64p,
                                 f64p, C.POINTER(CgConfig), f64p]),
    "gmrf_partition_owners": (C.c_int, [vp, C.c_int32, i32p]),
    "gmrf_partition_schedule": (C.c_int, [vp, i32p, i64p, i64p]),
    "gmrf_partition_memory": (C.c_int, [vp, C.c_int32, i32p, i64p]),
    "gmrf_factor_set_selinv_inplace": (C.c_int, [vp, C.c_int32]),
    "gmrf_factor_create_partitioned": (C.c_int, [vp, C.c_int32, C.c_int32, i32p, EXCHANGE_FN, vp,
                                                 C.POINTER(vp)]),
    "gmrf_spacetime_create_partitioned": (C.c_int, [C.POINTER(SpaceTimeConfig), C.c_int32,
                                                    C.c_int32, EXCHANGE_FN, vp, C.POINTER(vp)]),
    "gmrf_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "gmrf_nccl_comm_create": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.POINTER(vp)]),
    "gmrf_nccl_comm_destroy": (None, [vp]),
    "gmrf_nccl_exchange": (EXCHANGE_FN, []),
    "gmrf_nccl_last_error": (C.c_char_p, []),
    "gmrf_spacetime_create": (C.c_int, [C.POINTER(SpaceTimeConfig), C.POINTER(vp)]),
    "gmrf_spacetime_run": (C.c_int, [vp, f64p, C.c_int32, f64p, f64p, C.POINTER(GnIter),
                                     C.c_int32, i32p, i32p]),
    "gmrf_spacetime_info": (C.c_int, [vp, C.POINTER(SpaceTimeInfo)]),
    "gmrf_spacetime_symbolic": (C.c_int, [C.POINTER(SpaceTimeConfig), C.POINTER(vp)]),
    "gmrf_spacetime_device_results": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "gmrf_spacetime_pattern": (C.c_int, [vp, i64p, i32p, f64p, f64p]),
    "gmrf_spacetime_residual": (C.c_int, [vp, f64p, f64p]),
    "gmrf_spacetime_jacobian_nnz": (C.c_int, [vp, i64p]),
    "gmrf_spacetime_jacobian": (C.c_int, [vp, f64p, i64p, i32p, f64p]),
    "gmrf_spacetime_free": (None, [vp]),
    "gmrf_spacetime_set_profile": (C.c_int, [vp, C.c_int32]),
    "gmrf_gram_create": (C.c_int, [vp, C.c_int32, i64p, i32p, C.POINTER(vp)]),
    "gmrf_update_system_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, i64p, i32p, f64p,
                                            C.c_int32, i64p, i32p, i32p, C.POINTER(vp)]),
    "gmrf_update_system_same_operator": (C.c_int, [vp, C.c_int32, i64p, i32p]),
    "gmrf_update_system_refactor": (C.c_int, [vp, f64p, f64p, i32p]),
    "gmrf_update_system_refactor_solve": (C.c_int, [vp, f64p, f64p, f64p, f64p, i32p]),
    "gmrf_update_system_matrix": (C.c_int, [vp, i64p, i32p, f64p]),
    "gmrf_update_system_assemble": (C.c_int, [vp, f64p, f64p, C.c_double, f64p]),
    "gmrf_update_system_symbolic": (vp, [vp]),
    "gmrf_update_system_factor": (vp, [vp]),
    "gmrf_update_system_free": (None, [vp]),
    "gmrf_gram_free": (None, [vp]),
    "gmrf_gram_apply": (C.c_int, [vp, f64p, f64p, f64p, C.c_double, f64p]),
    "gmrf_factor_update_fixed_pattern": (C.c_int, [vp, vp, f64p, f64p, f64p, C.c_double, i32p]),
    "gmrf_factor_update_fixed_pattern_device": (C.c_int, [vp, vp, vp, vp, vp, C.c_double, i32p]),
    "gmrf_point_operator": (C.c_int, [C.POINTER(MaternConfig), C.c_int32, f64p, i64p, i32p,
                                      f64p]),
    "gmrf_matern_prior": (C.c_int, [C.POINTER(MaternConfig), i32p, i64p, i32p, f64p]),
    "gmrf_fem_assemble": (C.c_int, [C.POINTER(MaternConfig), C.c_int32, C.c_double, C.c_double,
                                    C.c_double, C.c_int32, C.c_double, i32p, i64p, i32p, f64p, f64p]),
    "gmrf_fem_assemble_host": (C.c_int, [C.POINTER(MaternConfig), C.c_int32, C.c_double, C.c_double,
                                         C.c_double, C.c_int32, C.c_double, i32p, i64p, i32p, f64p,
                                         f64p]),
    "gmrf_regression_create": (C.c_int, [C.POINTER(MaternConfig), C.c_int32, f64p, i32p,
                                         C.POINTER(vp)]),
    "gmrf_regression_run": (C.c_int, [vp, f64p, f64p, C.c_int32, C.c_int32, C.c_uint64, f64p,
                                      f64p, f64p]),
    "gmrf_regression_info": (C.c_int, [vp, C.POINTER(RegressionInfo)]),
    "gmrf_regression_precisions": (C.c_int, [vp, i64p, i32p, f64p, f64p]),
    "gmrf_regression_factor": (vp, [vp]),
    "gmrf_regression_free": (None, [vp]),
    "gmrf_spacetime_kernel_stats": (C.c_int, [vp, C.c_void_p, C.c_int32, i32p]),
}


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_int64), ("ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]

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
