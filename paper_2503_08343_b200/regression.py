"""Matérn SPDE regression posterior (configs 1-2): host mirror of the
reference's linear chain

    matern_prior(space, spec)                         priors/matern.hpp:53-80
    point_observation_operator(space, points, y, Λ)   solver/info_operator.hpp:108-123
    condition_on(prior, op)                           gmrf.hpp:145-170
    variance_takahashi(post), sample_direct(post, rng) gmrf.hpp:173-207

over the C-ABI pipeline ``gmrf_regression_*`` (include/gmrf_b200.h): prior
assembly, the fixed-pattern update Q + AᵀΛA (written straight into the factor
storage), factorization, mean solve, selected-inversion variances and samples
all run on the device. Point location (m points) is host work; there is no CPU
compute path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import f64p, i32p, i64p, ptr
from .core import SparseMatrixCSC, _check


@dataclass
class Mesh:
    """dim 1: build_interval_mesh(n_el, xa, xb) (fem/mesh.hpp:63); dim 2:
    build_unit_square_mesh(n_el) (mesh.hpp:142)."""
    dim: int = 1
    n_el: int = 999
    xa: float = 0.0
    xb: float = 1.0

    @staticmethod
    def interval(n_el, a=0.0, b=1.0) -> "Mesh":
        return Mesh(1, n_el, a, b)

    @staticmethod
    def unit_square(n_per_dim) -> "Mesh":
        return Mesh(2, n_per_dim, 0.0, 1.0)

    @property
    def n_dofs(self) -> int:
        return (self.n_el + 1) ** self.dim


@dataclass
class MaternSpec:
    """priors/matern.hpp MaternSpec {κ, α, τ}."""
    kappa: float = 1.0
    alpha: int = 2
    tau: float = 1.0


def _cfg(mesh: Mesh, spec: MaternSpec | None = None) -> _capi.MaternConfig:
    spec = spec or MaternSpec()
    return _capi.MaternConfig(mesh.dim, mesh.n_el, mesh.xa, mesh.xb, spec.kappa, spec.alpha,
                              spec.tau)


def point_observation_operator(mesh: Mesh, points) -> SparseMatrixCSC:
    """A_ij = φ_j(x_i) for P1 (eval_basis, fem/space.hpp:376-394); returned as a
    CSC m × n like the reference (built from the library's CSR)."""
    pts = np.ascontiguousarray(points, np.float64).ravel()
    m = len(pts) // mesh.dim
    c = _cfg(mesh)
    lib = _capi.load()
    rp = np.empty(m + 1, np.int64)
    _check(lib.gmrf_point_operator(C.byref(c), m, ptr(pts, f64p), ptr(rp, i64p), None, None))
    ci = np.empty(rp[-1], np.int32)
    v = np.empty(rp[-1], np.float64)
    _check(lib.gmrf_point_operator(C.byref(c), m, ptr(pts, f64p), ptr(rp, i64p), ptr(ci, i32p),
                                   ptr(v, f64p)))
    import scipy.sparse as sp
    a = sp.csr_matrix((v, ci, rp), shape=(m, mesh.n_dofs)).tocsc()
    a.sort_indices()
    return SparseMatrixCSC.from_scipy(a)


def matern_prior(mesh: Mesh, spec: MaternSpec) -> SparseMatrixCSC:
    """Prior precision Q (priors/matern.hpp:53-80), assembled on the device."""
    c = _cfg(mesh, spec)
    lib = _capi.load()
    n = C.c_int32()
    cp = np.empty(mesh.n_dofs + 1, np.int64)
    _check(lib.gmrf_matern_prior(C.byref(c), C.byref(n), ptr(cp, i64p), None, None))
    ri = np.empty(cp[-1], np.int32)
    v = np.empty(cp[-1], np.float64)
    _check(lib.gmrf_matern_prior(C.byref(c), C.byref(n), ptr(cp, i64p), ptr(ri, i32p),
                                 ptr(v, f64p)))
    return SparseMatrixCSC(n.value, n.value, cp, ri, v)


class RegressionPosterior:
    """condition_on(matern_prior(mesh, spec), point_observation_operator(mesh,
    points, ·, Λ)) on the device. perm: factor ordering (new -> old) or None for
    nested dissection (pass the reference's AMD order to reproduce its samples)."""

    def __init__(self, mesh: Mesh, spec: MaternSpec, points, perm=None):
        self.mesh, self.spec = mesh, spec
        self.points = np.ascontiguousarray(points, np.float64).ravel()
        self.m = len(self.points) // mesh.dim
        c = _cfg(mesh, spec)
        lib = _capi.load()
        h = C.c_void_p()
        pm = None if perm is None else np.ascontiguousarray(perm, np.int32)
        _check(lib.gmrf_regression_create(C.byref(c), self.m, ptr(self.points, f64p),
                                          ptr(pm, i32p), C.byref(h)))
        self._h = h
        self.n = self.info().n

    def __del__(self):
        if getattr(self, "_h", None):
            _capi.load().gmrf_regression_free(self._h)
            self._h = None

    def info(self) -> _capi.RegressionInfo:
        i = _capi.RegressionInfo()
        _check(_capi.load().gmrf_regression_info(self._h, C.byref(i)))
        return i

    def run(self, y, noise_prec, variances=True, n_samples=0, seed=0):
        """Returns (mean, var or None, samples n × n_samples or None)."""
        y = np.ascontiguousarray(y, np.float64)
        lam = np.ascontiguousarray(np.broadcast_to(noise_prec, (self.m,)), np.float64)
        mean = np.empty(self.n)
        var = np.empty(self.n) if variances else None
        smp = np.empty((n_samples, self.n)) if n_samples > 0 else None
        _check(_capi.load().gmrf_regression_run(self._h, ptr(y, f64p), ptr(lam, f64p),
                                                int(variances), int(n_samples), int(seed),
                                                ptr(mean, f64p), ptr(var, f64p), ptr(smp, f64p)))
        return mean, var, (None if smp is None else smp.T)

    def precisions(self):
        """(pattern col_ptr, row_idx, Q_prior values, Q_post values) — tests."""
        i = self.info()
        cp = np.empty(self.n + 1, np.int64)
        ri = np.empty(i.nnz_pattern, np.int32)
        qa = np.empty(i.nnz_pattern)
        qb = np.empty(i.nnz_pattern)
        _check(_capi.load().gmrf_regression_precisions(self._h, ptr(cp, i64p), ptr(ri, i32p),
                                                       ptr(qa, f64p), ptr(qb, f64p)))
        return cp, ri, qa, qb


def seeded_inputs(config: int):
    """SURVEY §8(d)'s pinned synthetic inputs for configs 1-2 (Rng = the
    reference's stream, core/rng.hpp): (mesh, spec, points, y, noise_prec,
    n_samples, sample_seed)."""
    from .core import Rng
    if config == 1:
        u, e = Rng(1001).draw(100, 100)
        y = np.sin(2 * np.pi * u) + 0.01 * e
        return Mesh.interval(999), MaternSpec(20.0, 2, 1.0), u, y, 1e4, 8, 2001
    if config == 2:
        u, e = Rng(1002).draw(4000, 2000)
        x, yy = u[0::2], u[1::2]
        y = np.sin(3 * np.pi * x) * np.cos(2 * np.pi * yy) + 0.05 * e
        return Mesh.unit_square(255), MaternSpec(10.0, 2, 1.0), u, y, 400.0, 16, 2002
    raise ValueError("configs 1 and 2 only")
