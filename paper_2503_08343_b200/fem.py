"""P1 finite-element matrices of one time slice: host
mirror of the reference's ``assemble_mass`` / ``assemble_stiffness``
(fem/assembly.hpp:81-161), ``lumped_mass_vector`` (:241-262) and the Dirichlet
``fold_and_mask`` (fem/constraints.hpp:111-128,158-173) over the C-ABI entry
``gmrf_fem_assemble`` (device kernels, csrc/fem_device.cu). ``device=False``
evaluates the same closed forms in host loops (``gmrf_fem_assemble_host``,
used by the CPU tests); the two agree bit for bit.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import f64p, i32p, i64p, ptr
from .core import SparseMatrixCSC, _check
from .regression import Mesh, MaternSpec, _cfg


def assemble_p1(mesh: Mesh, which: str, diffusion: float = 1.0, advection: float = 0.0,
                reaction: float = 0.0, dirichlet: bool = False, constrained_diag: float = 1.0,
                lumped: bool = False, device: bool = True):
    """which: "mass" or "stiffness". Returns the full CSC matrix, and the lumped
    row sums as well when ``lumped`` is set."""
    k = {"mass": 0, "stiffness": 1}[which]
    c = _cfg(mesh, MaternSpec())
    lib = _capi.load()
    fn = lib.gmrf_fem_assemble if device else lib.gmrf_fem_assemble_host
    n = C.c_int32()
    cp = np.empty(mesh.n_dofs + 1, np.int64)
    args = (C.byref(c), k, diffusion, advection, reaction, int(dirichlet), constrained_diag,
            C.byref(n), ptr(cp, i64p))
    _check(fn(*args, None, None, None))
    ri = np.empty(cp[-1], np.int32)
    v = np.empty(cp[-1], np.float64)
    lum = np.empty(mesh.n_dofs) if lumped else None
    _check(fn(*args, ptr(ri, i32p), ptr(v, f64p), ptr(lum, f64p)))
    m = SparseMatrixCSC(n.value, n.value, cp, ri, v)
    return (m, lum) if lumped else m
