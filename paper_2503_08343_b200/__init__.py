"""B200-native sparse-precision GMRF inference engine (arXiv 2503.08343 hot path).

The compute path is libgmrf_b200.so (include/gmrf_b200.h): host symbolic
analysis in C++ and sm_100a CUDA kernels for the supernodal Cholesky
factorization, triangular solves and selected inversion. This package is the
host-side mirror of the reference API (gmrfpde core/*).
"""
from .core import (  # noqa: F401
    CGConfig,
    CGResult,
    Preconditioner,
    Rng,
    cg_solve,
    sample_cg,
    CholeskyFactor,
    ContractError,
    DeviceError,
    DimensionError,
    NotPositiveDefiniteError,
    NumericalError,
    SparseMatrixCSC,
    StructuralError,
    SymbolicFactor,
    TriangularMode,
    bench_fp64,
    cholesky_factor,
    cholesky_refactor,
    nd_order,
    rbmc_variance,
    sample_direct,
    solve,
    solve_triangular,
    symbolic_analyze,
    takahashi_diagonal,
    takahashi_selected_inverse,
)
