"""Space-time GMRF posterior (configs 3-5): host mirror of the reference's
run_burgers chain (bench/runner.hpp:457-632) over the C-ABI pipeline
``gmrf_spacetime_*`` (include/gmrf_b200.h).

    spatiotemporal_prior  → condition_on(IC) → gauss_newton(residual)
    → laplace_posterior → variance_takahashi

residual: Burgers weak form (config 4, 1-D), or the Allen-Cahn weak form
(config 5, 2-D unit square; restated in oracle/ref_capi.cpp since the reference
has no Allen-Cahn residual).

Everything after the host-side spatial blocks and symbolic analysis runs on
the device; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import f64p, i32p, i64p, ptr
from .core import NumericalError, _check


@dataclass
class MaternSpec:
    kappa: float = 1.0
    alpha: int = 2
    tau: float = 1.0


@dataclass
class GaussNewtonConfig:
    """gauss_newton.hpp:19-24."""
    max_iters: int = 10
    decrement_tol: float = 1e-5
    armijo_c: float = 1e-4
    shrink: float = 0.5
    max_backtracks: int = 30


@dataclass
class SpaceTimeSpec:
    n_el: int = 999
    xa: float = -1.0
    xb: float = 1.0
    n_t: int = 1000
    t_end: float = 1.0
    diffusion: float = 0.01 / math.pi
    advection: float = 0.5
    noise: MaternSpec = field(default_factory=lambda: MaternSpec(10.0, 1, 1.0))
    init: MaternSpec = field(default_factory=lambda: MaternSpec(10.0, 2, 1.0))
    tau: float = 1.0
    eps: float = 1e-10
    dirichlet: bool = True
    ic_noise_prec: float = 1e8
    residual: int = 1
    pde_noise_prec: float = 1e12
    dim: int = 1

    @staticmethod
    def burgers(n_el=999, n_t=1000) -> "SpaceTimeSpec":
        """Config 4."""
        return SpaceTimeSpec(n_el=n_el, n_t=n_t)

    @staticmethod
    def heat(n_el=499, n_t=1000) -> "SpaceTimeSpec":
        """Config 3."""
        return SpaceTimeSpec(n_el=n_el, xa=0.0, xb=1.0, n_t=n_t, diffusion=0.1, advection=0.0,
                             ic_noise_prec=1e6, residual=0)

    @staticmethod
    def allen_cahn(n_cells=127, n_t=256) -> "SpaceTimeSpec":
        """Config 5: 128² unit-square P1 nodes × 256 slices over
        [0, 0.5], heat proxy laplace_operator(ε² = 0.0025), natural BC, IC Λ = 1e6,
        Allen-Cahn residual with Λ_pde = 1e12 (GN 8 steps)."""
        return SpaceTimeSpec(n_el=n_cells, xa=0.0, xb=1.0, n_t=n_t, t_end=0.5, diffusion=0.0025,
                             advection=0.0, dirichlet=False, ic_noise_prec=1e6, residual=2, dim=2)

    @property
    def n_space(self) -> int:
        return (self.n_el + 1) ** self.dim

    def node_xy(self) -> np.ndarray:
        """2-D node coordinates, DoF iy·(n+1) + ix (mesh.hpp:118-131)."""
        a = np.arange(self.n_el + 1) / self.n_el
        x, y = np.meshgrid(a, a)
        return np.stack([x.ravel(), y.ravel()], axis=1)

    def node_x(self) -> np.ndarray:
        i = np.arange(self.n_el + 1)
        x = self.xa + (self.xb - self.xa) * i / self.n_el
        x[-1] = self.xb
        return x


@dataclass
class GaussNewtonIteration:
    iter: int
    objective: float
    decrement: float
    step_size: float
    backtracks: int


class GaussNewtonStagnation(NumericalError):
    def __init__(self, msg, trace):
        super().__init__(msg)
        self._trace = trace

    def trace(self):
        return self._trace


def _config(spec: "SpaceTimeSpec", gn: "GaussNewtonConfig | None" = None):
    gn = gn or GaussNewtonConfig()
    return _capi.SpaceTimeConfig(
        spec.n_el, spec.xa, spec.xb, spec.n_t, spec.t_end, spec.diffusion, spec.advection,
        spec.noise.kappa, spec.noise.alpha, spec.noise.tau, spec.init.kappa, spec.init.alpha,
        spec.init.tau, spec.tau, spec.eps, int(spec.dirichlet), spec.ic_noise_prec,
        spec.residual, spec.pde_noise_prec, gn.max_iters, gn.decrement_tol, gn.armijo_c,
        gn.shrink, gn.max_backtracks, spec.dim)


def host_symbolic(spec: "SpaceTimeSpec"):
    """The pipeline factor's symbolic analysis on the host only (no device):
    returns (info, supernodes) with supernodes = dict(first, rows, level, parent)."""
    lib = _capi.load()
    c = _config(spec)
    h = C.c_void_p()
    _check(lib.gmrf_spacetime_symbolic(C.byref(c), C.byref(h)))
    try:
        info = _capi.SymbolicInfo()
        _check(lib.gmrf_symbolic_info(h, C.byref(info)))
        ns = info.n_supernodes
        first = np.empty(ns + 1, np.int32)
        rows, level, parent = (np.empty(ns, np.int32) for _ in range(3))
        _check(lib.gmrf_symbolic_supernodes(h, ptr(first, i32p), ptr(rows, i32p),
                                            ptr(level, i32p), ptr(parent, i32p)))
        return info, dict(first=first, rows=rows, level=level, parent=parent)
    finally:
        lib.gmrf_symbolic_free(h)


class SpaceTimePosterior:
    def __init__(self, spec: SpaceTimeSpec, gn: GaussNewtonConfig | None = None,
                 partition=None):
        """partition: None (whole problem on this GPU) or (nranks, rank, exchange)
        with an ``Exchange`` from paper_2503_08343_b200.partition — this rank's
        share of an ND-partitioned factorization; every rank gets the complete
        posterior."""
        gn = gn or GaussNewtonConfig()
        c = _capi.SpaceTimeConfig(
            spec.n_el, spec.xa, spec.xb, spec.n_t, spec.t_end, spec.diffusion, spec.advection,
            spec.noise.kappa, spec.noise.alpha, spec.noise.tau, spec.init.kappa, spec.init.alpha,
            spec.init.tau, spec.tau, spec.eps, int(spec.dirichlet), spec.ic_noise_prec,
            spec.residual, spec.pde_noise_prec, gn.max_iters, gn.decrement_tol, gn.armijo_c,
            gn.shrink, gn.max_backtracks, spec.dim)
        self.spec = spec
        lib = _capi.load()
        h = C.c_void_p()
        if partition is None:
            _check(lib.gmrf_spacetime_create(C.byref(c), C.byref(h)))
        else:
            nranks, rank, exchange = partition
            self._exchange = exchange  # the C callback must outlive the handle
            _check(lib.gmrf_spacetime_create_partitioned(C.byref(c), nranks, rank, exchange.fn,
                                                         getattr(exchange, "ctx", None),
                                                         C.byref(h)))
        self._h = h
        self.n = self.info().n

    def __del__(self):
        if getattr(self, "_h", None):
            _capi.load().gmrf_spacetime_free(self._h)
            self._h = None

    def info(self) -> _capi.SpaceTimeInfo:
        i = _capi.SpaceTimeInfo()
        _check(_capi.load().gmrf_spacetime_info(self._h, C.byref(i)))
        return i

    def run(self, u0, variances=True, copy_back=True, max_trace=64):
        """Returns (mean, var, trace, converged); mean/var None if copy_back is False."""
        u0 = np.ascontiguousarray(u0, np.float64)
        mean = np.empty(self.n) if copy_back else None
        var = np.empty(self.n) if (copy_back and variances) else None
        tr = (_capi.GnIter * max_trace)()
        nt, conv = C.c_int32(), C.c_int32()
        rc = _capi.load().gmrf_spacetime_run(self._h, ptr(u0, f64p), int(variances),
                                             ptr(mean, f64p), ptr(var, f64p), tr, max_trace,
                                             C.byref(nt), C.byref(conv))
        trace = [GaussNewtonIteration(t.iter, t.objective, t.decrement, t.step_size, t.backtracks)
                 for t in tr[: nt.value]]
        if rc == 6 and trace:
            raise GaussNewtonStagnation(_capi.load().gmrf_last_error().decode(), trace)
        _check(rc)
        return mean, var, trace, bool(conv.value)

    def set_profile(self, on: bool):
        _check(_capi.load().gmrf_spacetime_set_profile(self._h, int(on)))

    def kernel_stats(self) -> dict:
        """{kernel class: dict(launches, ms, flops, bytes)} accumulated since set_profile(True)."""
        arr = (_capi.KernelStat * 4096)()
        n = C.c_int32()
        _check(_capi.load().gmrf_spacetime_kernel_stats(self._h, C.cast(arr, C.c_void_p), 4096,
                                                        C.byref(n)))
        return {a.name.decode(): dict(launches=a.launches, ms=a.ms, flops=a.flops, bytes=a.bytes)
                for a in arr[: n.value]}

    def device_results(self):
        m, v = C.c_void_p(), C.c_void_p()
        _check(_capi.load().gmrf_spacetime_device_results(self._h, C.byref(m), C.byref(v)))
        return m.value, v.value

    def pattern(self):
        i = self.info()
        cp = np.empty(self.n + 1, np.int64)
        ri = np.empty(i.nnz_pattern, np.int32)
        qc = np.empty(i.nnz_pattern)
        qe = np.empty(i.nnz_pattern)
        _check(_capi.load().gmrf_spacetime_pattern(self._h, ptr(cp, i64p), ptr(ri, i32p),
                                                   ptr(qc, f64p), ptr(qe, f64p)))
        return cp, ri, qc, qe

    def residual(self, u):
        u = np.ascontiguousarray(u, np.float64)
        f = np.empty(self.info().n_res)
        _check(_capi.load().gmrf_spacetime_residual(self._h, ptr(u, f64p), ptr(f, f64p)))
        return f

    def jacobian(self, u):
        u = np.ascontiguousarray(u, np.float64)
        nnz = C.c_int64()
        _check(_capi.load().gmrf_spacetime_jacobian_nnz(self._h, C.byref(nnz)))
        nr = self.info().n_res
        rp = np.empty(nr + 1, np.int64)
        ci = np.empty(nnz.value, np.int32)
        v = np.empty(nnz.value)
        _check(_capi.load().gmrf_spacetime_jacobian(self._h, ptr(u, f64p), ptr(rp, i64p),
                                                    ptr(ci, i32p), ptr(v, f64p)))
        return rp, ci, v
