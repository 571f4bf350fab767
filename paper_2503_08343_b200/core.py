"""Host mirror of the reference's factorization API (gmrfpde core/*).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/gmrfpde/core/{cholesky,takahashi,types}.hpp, so
parity tests read like the reference's own tests. Every compute call goes
through the C-ABI (include/gmrf_b200.h) into the sm_100a kernels; there is no
CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import f64p, i32p, i64p, ptr


# ---- exception hierarchy (core/types.hpp:16-48) ----------------------------
class StructuralError(RuntimeError):
    pass


class DimensionError(StructuralError):
    pass


class ContractError(RuntimeError):
    pass


class NumericalError(RuntimeError):
    pass


class NotPositiveDefiniteError(NumericalError):
    """Carries the offending index in the ORIGINAL numbering (types.hpp:40-48)."""

    def __init__(self, msg: str, index: int):
        super().__init__(msg)
        self._index = int(index)

    def index(self) -> int:
        return self._index


class DeviceError(RuntimeError):
    pass


_ERRS = {1: NumericalError, 2: DimensionError, 3: StructuralError, 4: ContractError,
         5: DeviceError, 6: NumericalError}


def _check(rc: int, bad: int | None = None):
    if rc == 0:
        return
    msg = _capi.load().gmrf_last_error().decode()
    if rc == 1:
        raise NotPositiveDefiniteError(msg, -1 if bad is None else bad)
    raise _ERRS.get(rc, RuntimeError)(msg)


# ---- sparse carrier (core/sparse.hpp:25-61, int64 column pointers) ---------
@dataclass
class SparseMatrixCSC:
    nrows: int
    ncols: int
    col_ptr: np.ndarray  # int64[ncols+1]
    row_idx: np.ndarray  # int32[nnz]
    values: np.ndarray   # float64[nnz]

    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    @staticmethod
    def from_scipy(m) -> "SparseMatrixCSC":
        m = m.tocsc()
        m.sort_indices()
        return SparseMatrixCSC(m.shape[0], m.shape[1], np.ascontiguousarray(m.indptr, np.int64),
                               np.ascontiguousarray(m.indices, np.int32),
                               np.ascontiguousarray(m.data, np.float64))

    @staticmethod
    def from_arrays(nrows, ncols, col_ptr, row_idx, values) -> "SparseMatrixCSC":
        return SparseMatrixCSC(int(nrows), int(ncols), np.ascontiguousarray(col_ptr, np.int64),
                               np.ascontiguousarray(row_idx, np.int32),
                               np.ascontiguousarray(values, np.float64))

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csc_matrix((self.values, self.row_idx, self.col_ptr),
                             shape=(self.nrows, self.ncols))

    def coeff(self, i: int, j: int) -> float:
        a, b = self.col_ptr[j], self.col_ptr[j + 1]
        k = np.searchsorted(self.row_idx[a:b], i)
        if k < b - a and self.row_idx[a + k] == i:
            return float(self.values[a + k])
        return 0.0


class TriangularMode:
    kLower = 0
    kUpper = 1
    kFull = 2


@dataclass
class SymbolicFactor:
    """symbolic_analyze result (cholesky.hpp:16-23) plus the device handle."""
    n: int
    perm: np.ndarray
    perm_inv: np.ndarray
    parent: np.ndarray
    col_ptr: np.ndarray
    nnz_L: int
    info: _capi.SymbolicInfo
    _h: C.c_void_p = field(repr=False, default=None)
    _pattern: tuple = field(repr=False, default=None)

    def __del__(self):
        if self._h:
            _capi.load().gmrf_symbolic_free(self._h)
            self._h = None


def _validate_square(q: SparseMatrixCSC, what: str):
    if q.nrows != q.ncols:
        raise DimensionError(f"{what}: matrix not square")


def nd_order(q: SparseMatrixCSC) -> np.ndarray:
    """METIS nested-dissection ordering (new -> old); replaces amd_order."""
    _validate_square(q, "nd_order")
    lib = _capi.load()
    perm = np.empty(q.nrows, np.int32)
    _check(lib.gmrf_nd_order(q.nrows, ptr(q.col_ptr, i64p), ptr(q.row_idx, i32p), ptr(perm, i32p)))
    return perm


def symbolic_analyze(q: SparseMatrixCSC, perm=None) -> SymbolicFactor:
    """cholesky.hpp:68. perm=None → nested dissection (the reference's AMD slot)."""
    _validate_square(q, "symbolic_analyze")
    lib = _capi.load()
    n = q.nrows
    p = None if perm is None else np.ascontiguousarray(perm, np.int32)
    if p is not None and p.shape[0] != n:
        raise DimensionError("symbolic_analyze: permutation length mismatch")
    h = C.c_void_p()
    _check(lib.gmrf_symbolic_analyze(n, ptr(q.col_ptr, i64p), ptr(q.row_idx, i32p),
                                     ptr(p, i32p), C.byref(h)))
    info = _capi.SymbolicInfo()
    _check(lib.gmrf_symbolic_info(h, C.byref(info)))
    perm_o = np.empty(n, np.int32)
    parent = np.empty(n, np.int32)
    cpl = np.empty(n + 1, np.int64)
    _check(lib.gmrf_symbolic_export(h, ptr(perm_o, i32p), ptr(parent, i32p), ptr(cpl, i64p)))
    pinv = np.empty(n, np.int32)
    pinv[perm_o] = np.arange(n, dtype=np.int32)
    return SymbolicFactor(n, perm_o, pinv, parent, cpl, int(info.nnz_l), info, h,
                          (q.col_ptr.copy(), q.row_idx.copy()))


class CholeskyFactor:
    """Device-resident factor; ``L`` materialises the reference layout on demand
    (cholesky.hpp:92-109 readers such as takahashi.hpp:20 read ``f.L``)."""

    def __init__(self, sym: SymbolicFactor):
        self.sym = sym
        lib = _capi.load()
        h = C.c_void_p()
        _check(lib.gmrf_factor_create(sym._h, C.byref(h)))
        self._h = h
        self.perm = sym.perm
        self.perm_inv = sym.perm_inv
        self._L = None

    def __del__(self):
        if getattr(self, "_h", None):
            _capi.load().gmrf_factor_free(self._h)
            self._h = None

    def dim(self) -> int:
        return self.sym.n

    def refactor(self, q_values: np.ndarray):
        lib = _capi.load()
        bad = C.c_int32(-1)
        v = np.ascontiguousarray(q_values, np.float64)
        rc = lib.gmrf_factor_numeric(self._h, ptr(v, f64p), C.byref(bad))
        self._L = None
        _check(rc, bad.value)

    def refactor_device(self, d_q_values_ptr: int):
        lib = _capi.load()
        bad = C.c_int32(-1)
        rc = lib.gmrf_factor_numeric_device(self._h, C.c_void_p(d_q_values_ptr), C.byref(bad))
        self._L = None
        _check(rc, bad.value)

    @property
    def L(self) -> SparseMatrixCSC:
        if self._L is None:
            n = self.sym.n
            nnz = self.sym.nnz_L
            cp = np.empty(n + 1, np.int64)
            ri = np.empty(nnz, np.int32)
            v = np.empty(nnz, np.float64)
            _check(_capi.load().gmrf_factor_l(self._h, ptr(cp, i64p), ptr(ri, i32p),
                                              ptr(v, f64p), None))
            self._L = SparseMatrixCSC(n, n, cp, ri, v)
        return self._L

    def apply_perm(self, x):
        return np.asarray(x)[self.perm]

    def apply_perm_inv(self, x):
        y = np.empty_like(np.asarray(x))
        y[self.perm] = x
        return y

    def set_stream(self, stream_ptr: int):
        _check(_capi.load().gmrf_factor_set_stream(self._h, C.c_void_p(stream_ptr)))

    def stats(self) -> _capi.FactorStats:
        st = _capi.FactorStats()
        _check(_capi.load().gmrf_factor_stats(self._h, C.byref(st)))
        return st


def cholesky_refactor(sym: SymbolicFactor, q: SparseMatrixCSC) -> CholeskyFactor:
    """cholesky.hpp:113 — numeric factorization on a precomputed pattern."""
    if q.nrows != sym.n or q.ncols != sym.n:
        raise DimensionError("cholesky_refactor: dimension mismatch")
    cp, ri = sym._pattern
    if q.col_ptr.shape != cp.shape or not np.array_equal(q.col_ptr, cp) or \
            not np.array_equal(q.row_idx, ri):
        raise StructuralError("cholesky_refactor: pattern differs from the symbolic analysis")
    f = CholeskyFactor(sym)
    f.refactor(q.values)
    return f


def cholesky_factor(q: SparseMatrixCSC, perm=None) -> CholeskyFactor:
    """cholesky.hpp:164 (given perm) / :170 (default ordering: ND instead of AMD)."""
    return cholesky_refactor(symbolic_analyze(q, perm), q)


def solve_triangular(f: CholeskyFactor, b, mode: int) -> np.ndarray:
    """cholesky.hpp:179. b may be (n,) or (n, nrhs)."""
    b = np.asarray(b, np.float64)
    n = f.dim()
    if b.shape[0] != n:
        raise DimensionError("solve_triangular: dimension mismatch")
    if mode not in (0, 1, 2):
        raise ContractError("solve_triangular: unknown mode")
    if n == 0:
        return b.copy()
    bb = np.asfortranarray(b.reshape(n, -1))
    x = np.empty_like(bb, order="F")
    _check(_capi.load().gmrf_solve(f._h, int(mode), bb.shape[1], ptr(bb, f64p), ptr(x, f64p)))
    return x.reshape(b.shape)


def solve(f: CholeskyFactor, b) -> np.ndarray:
    """cholesky.hpp:225."""
    return solve_triangular(f, b, TriangularMode.kFull)


def takahashi_diagonal(f: CholeskyFactor) -> np.ndarray:
    """takahashi.hpp:67 — diag(Q⁻¹) in original order (supernodal selected inversion)."""
    d = np.empty(f.dim(), np.float64)
    _check(_capi.load().gmrf_selinv_diag(f._h, ptr(d, f64p)))
    return d


def sample_direct(f: CholeskyFactor, mean, n_samples: int, seed: int) -> np.ndarray:
    """gmrf.hpp:173/182 — ``n_samples`` draws μ + Pᵀ L⁻ᵀ z from one Rng(seed)
    stream (the reference's draw order); returns (n, n_samples)."""
    n = f.dim()
    mu = np.ascontiguousarray(mean, np.float64)
    if mu.shape[0] != n:
        raise DimensionError("sample_direct: mean length mismatch")
    out = np.empty((n, int(n_samples)), order="F")
    _check(_capi.load().gmrf_sample_direct(f._h, ptr(mu, f64p), int(n_samples), int(seed),
                                           ptr(out, f64p)))
    return out


def rbmc_variance(f: CholeskyFactor, q: SparseMatrixCSC, mean, n_samples: int,
                  seed: int) -> np.ndarray:
    """gmrf.hpp:213-240 — Rao-Blackwellized Monte Carlo marginal variances of
    N(mean, Q⁻¹) (f = the factor of q)."""
    n = f.dim()
    mu = np.ascontiguousarray(mean, np.float64)
    if mu.shape[0] != n or q.nrows != n:
        raise DimensionError("rbmc_variance: dimension mismatch")
    qv = np.ascontiguousarray(q.values, np.float64)
    var = np.empty(n)
    _check(_capi.load().gmrf_rbmc_variance(f._h, ptr(qv, f64p), ptr(mu, f64p), int(n_samples),
                                           int(seed), ptr(var, f64p)))
    return var


class Preconditioner:
    kNone = 0
    kJacobi = 1


@dataclass
class CGConfig:
    """cg.hpp:14-25."""
    rtol: float = 1e-8
    atol: float = 0.0
    max_iter: int = 0
    preconditioner: int = Preconditioner.kNone

    def _c(self):
        return _capi.CgConfig(self.rtol, self.atol, self.max_iter, self.preconditioner)


@dataclass
class CGResult:
    """cg.hpp:29-34."""
    x: np.ndarray
    iterations: int
    final_residual: float
    converged: bool


def cg_solve(q: SparseMatrixCSC, b, x0=None, cfg: CGConfig | None = None) -> CGResult:
    """cg.hpp:98 (matrix-backed cg_solve) on the device."""
    cfg = cfg or CGConfig()
    _validate_square(q, "cg_solve")
    n = q.nrows
    bb = np.ascontiguousarray(b, np.float64)
    if bb.shape[0] != n:
        raise DimensionError("cg: b dimension mismatch")
    xx0 = None if x0 is None or len(x0) == 0 else np.ascontiguousarray(x0, np.float64)
    if xx0 is not None and xx0.shape[0] != n:
        raise DimensionError("cg: x0 dimension mismatch")
    x = np.empty(n)
    r = _capi.CgResult()
    c = cfg._c()
    _check(_capi.load().gmrf_cg_solve(n, ptr(q.col_ptr, i64p), ptr(q.row_idx, i32p),
                                      ptr(q.values, f64p), ptr(bb, f64p), ptr(xx0, f64p),
                                      C.byref(c), ptr(x, f64p), C.byref(r)))
    return CGResult(x, int(r.iterations), float(r.final_residual), bool(r.converged))


def sample_cg(q: SparseMatrixCSC, s: SparseMatrixCSC, mean, z, cfg: CGConfig | None = None):
    """gmrf.hpp:188 — mean + Q⁻¹ S z by CG (S = the square root, n × m)."""
    cfg = cfg or CGConfig()
    n = q.nrows
    zz = np.ascontiguousarray(z, np.float64)
    if zz.shape[0] != s.ncols:
        raise DimensionError("sample_cg: z length must equal sqrt column count")
    mu = np.ascontiguousarray(mean, np.float64)
    out = np.empty(n)
    c = cfg._c()
    _check(_capi.load().gmrf_sample_cg(n, ptr(q.col_ptr, i64p), ptr(q.row_idx, i32p),
                                       ptr(q.values, f64p), s.ncols, ptr(s.col_ptr, i64p),
                                       ptr(s.row_idx, i32p), ptr(s.values, f64p), ptr(mu, f64p),
                                       ptr(zz, f64p), C.byref(c), ptr(out, f64p)))
    return out


def takahashi_selected_inverse(f: CholeskyFactor) -> SparseMatrixCSC:
    """takahashi.hpp:19 — Σ on the pattern of L+Lᵀ, original indices."""
    lib = _capi.load()
    takahashi_diagonal(f)
    nnz = C.c_int64()
    _check(lib.gmrf_selinv_pattern_nnz(f._h, C.byref(nnz)))
    n = f.dim()
    cp = np.empty(n + 1, np.int64)
    ri = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    _check(lib.gmrf_selinv_pattern(f._h, ptr(cp, i64p), ptr(ri, i32p), ptr(v, f64p)))
    return SparseMatrixCSC(n, n, cp, ri, v)


class Rng:
    """core/rng.hpp:14-47 draws (mt19937_64 + Box-Muller with a cached spare),
    generated in the library (host); the stream restarts per call."""

    def __init__(self, seed: int):
        self.seed = int(seed)

    def _fill(self, kind, n):
        out = np.empty(int(n))
        _check(_capi.load().gmrf_rng_fill(self.seed, kind, int(n), ptr(out, f64p)))
        return out

    def uniforms(self, n):
        """The first n values of uniform() from a fresh Rng(seed)."""
        return self._fill(0, n)

    def normal_vector(self, n):
        """normal_vector(n) of a fresh Rng(seed)."""
        return self._fill(1, n)

    def draw(self, n_uniform, n_normal):
        """One fresh Rng(seed) stream: n_uniform uniform() then n_normal normal()."""
        out = np.empty(int(n_uniform) + int(n_normal))
        _check(_capi.load().gmrf_rng_draw(self.seed, int(n_uniform), int(n_normal),
                                          ptr(out, f64p)))
        return out[: int(n_uniform)], out[int(n_uniform):]


def bench_fp64() -> tuple[float, float]:
    a, b = C.c_double(), C.c_double()
    _check(_capi.load().gmrf_bench_fp64(C.byref(a), C.byref(b)))
    return a.value, b.value
