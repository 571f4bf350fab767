"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes access to the two CPU checkers built by oracle/Makefile:
  * ``Port``  — oracle/_build/liboracle.so, our C restatement (gmrf_oracle.c);
  * ``Ref``   — oracle/_ref/libgmrfref.so, the unmodified reference headers
                compiled through oracle/ref_capi.cpp (absent when the reference
                was not available at build time).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgmrfref.so")
REF_ND_SO = os.path.join(HERE, "_ref", "libgmrfref_nd.so")
# the same reference chains compiled against the drop-in headers (the B200 engine
# behind the reference API); not a checker — what tests/test_gpu_dropin.py checks
REF_B200_SO = os.path.join(HERE, "_ref", "libgmrfref_b200.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Port:
    """C restatement of core/cholesky.hpp + core/takahashi.hpp (int64 col_ptr)."""

    def __init__(self):
        if not os.path.exists(PORT_SO):
            build()
        lib = C.CDLL(PORT_SO)
        lib.orc_symbolic.argtypes = [C.c_int32, i64p, i32p, i32p, i32p, i64p]
        lib.orc_cholesky.restype = C.c_int32
        lib.orc_cholesky.argtypes = [C.c_int32, i64p, i32p, f64p, i32p, i64p, i32p, f64p]
        lib.orc_solve.argtypes = [C.c_int32, i64p, i32p, f64p, i32p, C.c_int, C.c_int32, f64p, f64p]
        lib.orc_takahashi.argtypes = [C.c_int32, i64p, i32p, f64p, f64p]
        lib.orc_takahashi_diag.argtypes = [C.c_int32, i64p, i32p, f64p, i32p, f64p]
        self.lib = lib

    def symbolic(self, n, cp, ri, perm):
        cp = np.ascontiguousarray(cp, np.int64)
        ri = np.ascontiguousarray(ri, np.int32)
        perm = np.ascontiguousarray(perm, np.int32)
        parent = np.empty(n, np.int32)
        cpl = np.empty(n + 1, np.int64)
        self.lib.orc_symbolic(n, _p(cp, i64p), _p(ri, i32p), _p(perm, i32p), _p(parent, i32p),
                              _p(cpl, i64p))
        return parent, cpl

    def cholesky(self, n, cp, ri, v, perm):
        """Returns (L col_ptr, row_idx, values, bad_original_index_or_-1)."""
        cp = np.ascontiguousarray(cp, np.int64)
        ri = np.ascontiguousarray(ri, np.int32)
        v = np.ascontiguousarray(v, np.float64)
        perm = np.ascontiguousarray(perm, np.int32)
        _, lcp = self.symbolic(n, cp, ri, perm)
        lri = np.zeros(lcp[-1], np.int32)
        lv = np.zeros(lcp[-1], np.float64)
        bad = self.lib.orc_cholesky(n, _p(cp, i64p), _p(ri, i32p), _p(v, f64p), _p(perm, i32p),
                                    _p(lcp, i64p), _p(lri, i32p), _p(lv, f64p))
        return lcp, lri, lv, int(bad)

    def solve(self, n, lcp, lri, lv, perm, mode, b):
        b = np.asfortranarray(np.asarray(b, np.float64).reshape(n, -1))
        x = np.empty_like(b, order="F")
        self.lib.orc_solve(n, _p(lcp, i64p), _p(lri, i32p), _p(lv, f64p),
                           _p(np.ascontiguousarray(perm, np.int32), i32p), mode, b.shape[1],
                           _p(b, f64p), _p(x, f64p))
        return x

    def takahashi(self, n, lcp, lri, lv):
        sv = np.empty(lcp[-1], np.float64)
        self.lib.orc_takahashi(n, _p(lcp, i64p), _p(lri, i32p), _p(lv, f64p), _p(sv, f64p))
        return sv

    def takahashi_diag(self, n, lcp, lri, lv, perm):
        out = np.empty(n, np.float64)
        self.lib.orc_takahashi_diag(n, _p(lcp, i64p), _p(lri, i32p), _p(lv, f64p),
                                    _p(np.ascontiguousarray(perm, np.int32), i32p), _p(out, f64p))
        return out


class RefMatrix:
    def __init__(self, nrows, ncols, cp, ri, v):
        self.nrows, self.ncols = nrows, ncols
        self.col_ptr, self.row_idx, self.values = cp, ri, v


class Ref:
    """The reference itself (int32 CSC, as core/types.hpp:12)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, so: str = REF_SO):
        """so: REF_SO, or REF_ND_SO — the ordering-floor probe build (the chain's AMD
        redirected to METIS nested dissection, oracle/ref_capi.cpp); load one per
        process."""
        lib = C.CDLL(so)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_build.restype = C.c_void_p
        lib.ref_build.argtypes = [C.c_char_p, f64p, C.c_int]
        lib.ref_bundle_free.argtypes = [C.c_void_p]
        lib.ref_bundle_mat_shape.argtypes = [C.c_void_p, C.c_char_p, i32p, i32p, i32p]
        lib.ref_bundle_mat_copy.argtypes = [C.c_void_p, C.c_char_p, i32p, i32p, f64p]
        lib.ref_bundle_vec_len.restype = C.c_longlong
        lib.ref_bundle_vec_len.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_bundle_vec_copy.argtypes = [C.c_void_p, C.c_char_p, f64p]
        lib.ref_bundle_scalar.restype = C.c_double
        lib.ref_bundle_scalar.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_amd_order.argtypes = [C.c_int, i32p, i32p, i32p]
        lib.ref_symbolic.argtypes = [C.c_int, i32p, i32p, i32p, i32p, i32p]
        lib.ref_factor.restype = C.c_void_p
        lib.ref_factor.argtypes = [C.c_int, i32p, i32p, f64p, i32p, i32p]
        lib.ref_factor_free.argtypes = [C.c_void_p]
        lib.ref_factor_nnz.argtypes = [C.c_void_p]
        lib.ref_factor_copy.argtypes = [C.c_void_p, i32p, i32p, f64p, i32p]
        lib.ref_solve.argtypes = [C.c_void_p, C.c_int, f64p, f64p]
        lib.ref_takahashi_diag.argtypes = [C.c_void_p, f64p]
        lib.ref_takahashi_full.restype = C.c_void_p
        lib.ref_takahashi_full.argtypes = [C.c_void_p]
        lib.ref_condition_affine.restype = C.c_void_p
        lib.ref_condition_affine.argtypes = [C.c_int, i32p, i32p, f64p, f64p, C.c_int, i32p, i32p,
                                             f64p, f64p, f64p, f64p]
        lib.ref_time_stages.argtypes = [C.c_int, i32p, i32p, f64p, C.c_int, f64p]
        lib.ref_cg_solve.argtypes = [C.c_int, i32p, i32p, f64p, f64p, C.c_double, C.c_double,
                                     C.c_longlong, C.c_int, f64p, f64p]
        for nm in ("ref_sample_direct", "ref_rbmc_variance"):
            getattr(lib, nm).argtypes = [C.c_int, i32p, i32p, f64p, i32p, f64p, C.c_int,
                                         C.c_ulonglong, f64p]
        self.lib = lib

    def err(self):
        return self.lib.ref_last_error().decode()

    # ---- bundles ----
    def build(self, kind, params):
        p = np.ascontiguousarray(params, np.float64)
        h = self.lib.ref_build(kind.encode(), _p(p, f64p), len(p))
        if not h:
            raise RuntimeError(self.err())
        return Bundle(self, h)

    # ---- linear algebra ----
    @staticmethod
    def _csc32(cp, ri, v=None):
        return (np.ascontiguousarray(cp, np.int32), np.ascontiguousarray(ri, np.int32),
                None if v is None else np.ascontiguousarray(v, np.float64))

    def amd_order(self, n, cp, ri):
        cp, ri, _ = self._csc32(cp, ri)
        perm = np.empty(n, np.int32)
        if self.lib.ref_amd_order(n, _p(cp, i32p), _p(ri, i32p), _p(perm, i32p)) != 0:
            raise RuntimeError(self.err())
        return perm

    def symbolic(self, n, cp, ri, perm):
        cp, ri, _ = self._csc32(cp, ri)
        perm = np.ascontiguousarray(perm, np.int32)
        parent = np.empty(n, np.int32)
        cpl = np.empty(n + 1, np.int32)
        if self.lib.ref_symbolic(n, _p(cp, i32p), _p(ri, i32p), _p(perm, i32p), _p(parent, i32p),
                                 _p(cpl, i32p)) != 0:
            raise RuntimeError(self.err())
        return parent, cpl

    def factor(self, n, cp, ri, v, perm=None):
        cp, ri, v = self._csc32(cp, ri, v)
        pp = None if perm is None else np.ascontiguousarray(perm, np.int32)
        bad = C.c_int32(-1)
        h = self.lib.ref_factor(n, _p(cp, i32p), _p(ri, i32p), _p(v, f64p), _p(pp, i32p),
                                C.byref(bad))
        return RefFactor(self, h, n, bad.value)

    def condition_affine(self, n, q, mu, a, b, y, noise):
        qcp, qri, qv = self._csc32(*q)
        acp, ari, av = self._csc32(*a)
        m = len(y)
        h = self.lib.ref_condition_affine(
            n, _p(qcp, i32p), _p(qri, i32p), _p(qv, f64p),
            _p(np.ascontiguousarray(mu, np.float64), f64p), m, _p(acp, i32p), _p(ari, i32p),
            _p(av, f64p), _p(np.ascontiguousarray(b, np.float64), f64p),
            _p(np.ascontiguousarray(y, np.float64), f64p),
            _p(np.ascontiguousarray(noise, np.float64), f64p))
        if not h:
            raise RuntimeError(self.err())
        return Bundle(self, h)

    def sample_direct(self, n, cp, ri, v, perm, mu, ns, seed):
        """ns draws of sample_direct(g, rng) (gmrf.hpp:182), factor in `perm`."""
        cp, ri, v = self._csc32(cp, ri, v)
        out = np.empty((n, ns), order="F")
        if self.lib.ref_sample_direct(n, _p(cp, i32p), _p(ri, i32p), _p(v, f64p),
                                      _p(np.ascontiguousarray(perm, np.int32), i32p),
                                      _p(np.ascontiguousarray(mu, np.float64), f64p), ns, seed,
                                      _p(out, f64p)) != 0:
            raise RuntimeError(self.err())
        return out

    def rbmc_variance(self, n, cp, ri, v, perm, mu, ns, seed):
        """rbmc_variance (gmrf.hpp:213), factor in `perm`."""
        cp, ri, v = self._csc32(cp, ri, v)
        out = np.empty(n)
        if self.lib.ref_rbmc_variance(n, _p(cp, i32p), _p(ri, i32p), _p(v, f64p),
                                      _p(np.ascontiguousarray(perm, np.int32), i32p),
                                      _p(np.ascontiguousarray(mu, np.float64), f64p), ns, seed,
                                      _p(out, f64p)) != 0:
            raise RuntimeError(self.err())
        return out

    def cg_solve(self, n, cp, ri, v, b, rtol=1e-8, atol=0.0, max_iter=0, jacobi=False):
        """cg_solve (cg.hpp:98) → (x, iterations, final_residual, converged)."""
        cp, ri, v = self._csc32(cp, ri, v)
        x = np.empty(n)
        info = np.zeros(3)
        if self.lib.ref_cg_solve(n, _p(cp, i32p), _p(ri, i32p), _p(v, f64p),
                                 _p(np.ascontiguousarray(b, np.float64), f64p), rtol, atol,
                                 max_iter, int(jacobi), _p(x, f64p), _p(info, f64p)) != 0:
            raise RuntimeError(self.err())
        return x, int(info[0]), float(info[1]), bool(info[2])

    def time_stages(self, n, cp, ri, v, do_taka):
        cp, ri, v = self._csc32(cp, ri, v)
        out = np.zeros(7, np.float64)
        if self.lib.ref_time_stages(n, _p(cp, i32p), _p(ri, i32p), _p(v, f64p), int(do_taka),
                                    _p(out, f64p)) != 0:
            raise RuntimeError(self.err())
        return dict(amd_s=out[0], symbolic_s=out[1], numeric_s=out[2], solve_s=out[3],
                    takahashi_s=out[4], nnz_l=out[5], flops=out[6])


class RefFactor:
    def __init__(self, ref, h, n, bad):
        self.ref, self.h, self.n, self.bad = ref, h, n, bad

    def ok(self):
        return bool(self.h)

    def __del__(self):
        if self.h:
            self.ref.lib.ref_factor_free(self.h)
            self.h = None

    def L(self):
        nnz = self.ref.lib.ref_factor_nnz(self.h)
        cp = np.empty(self.n + 1, np.int32)
        ri = np.empty(nnz, np.int32)
        v = np.empty(nnz, np.float64)
        perm = np.empty(self.n, np.int32)
        self.ref.lib.ref_factor_copy(self.h, _p(cp, i32p), _p(ri, i32p), _p(v, f64p),
                                     _p(perm, i32p))
        return cp.astype(np.int64), ri, v, perm

    def solve(self, mode, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        self.ref.lib.ref_solve(self.h, mode, _p(b, f64p), _p(x, f64p))
        return x

    def takahashi_diag(self):
        out = np.empty(self.n, np.float64)
        self.ref.lib.ref_takahashi_diag(self.h, _p(out, f64p))
        return out

    def takahashi_full(self):
        b = Bundle(self.ref, self.ref.lib.ref_takahashi_full(self.h))
        return b.mat("S")


class Bundle:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        if self.h:
            self.ref.lib.ref_bundle_free(self.h)
            self.h = None

    def mat(self, name):
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int()
        if self.ref.lib.ref_bundle_mat_shape(self.h, name.encode(), C.byref(nr), C.byref(nc),
                                             C.byref(nnz)) != 0:
            raise KeyError(name)
        cp = np.empty(nc.value + 1, np.int32)
        ri = np.empty(nnz.value, np.int32)
        v = np.empty(nnz.value, np.float64)
        self.ref.lib.ref_bundle_mat_copy(self.h, name.encode(), _p(cp, i32p), _p(ri, i32p),
                                         _p(v, f64p))
        return RefMatrix(nr.value, nc.value, cp.astype(np.int64), ri, v)

    def vec(self, name):
        ln = self.ref.lib.ref_bundle_vec_len(self.h, name.encode())
        if ln == -1:
            raise KeyError(name)
        is_int = ln <= -2
        n = -2 - ln if is_int else ln
        out = np.empty(n, np.float64)
        self.ref.lib.ref_bundle_vec_copy(self.h, name.encode(), _p(out, f64p))
        return out.astype(np.int64) if is_int else out

    def scalar(self, name):
        return self.ref.lib.ref_bundle_scalar(self.h, name.encode())
