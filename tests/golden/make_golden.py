"""Generates the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libgmrfref.so, which compiles the
unmodified /root/reference headers):  python tests/golden/make_golden.py

Each fixture is the reference's output on seeded inputs (the reference ships no
golden files). The GPU box has no /root/reference, so tests
there read these .npz files.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Ref  # noqa: E402


def mat(prefix, m):
    return {f"{prefix}_cp": m.col_ptr, f"{prefix}_ri": m.row_idx, f"{prefix}_v": m.values,
            f"{prefix}_shape": np.array([m.nrows, m.ncols])}


def corpus(ref, count, seed, name):
    """spd_corpus (tests/oracles.hpp:208-284) + reference factor/solve/Takahashi."""
    b = ref.build("corpus", [count, seed])
    out = {}
    rng = np.random.default_rng(seed)
    for i in range(count):
        q = b.mat(f"Q{i}")
        n = q.nrows
        perm = ref.amd_order(n, q.col_ptr, q.row_idx)
        f = ref.factor(n, q.col_ptr, q.row_idx, q.values, perm)
        lcp, lri, lv, _ = f.L()
        rhs = rng.standard_normal(n)
        out.update(mat(f"Q{i}", q))
        out[f"perm{i}"] = perm
        out[f"L{i}_cp"], out[f"L{i}_ri"], out[f"L{i}_v"] = lcp, lri, lv
        out[f"b{i}"] = rhs
        out[f"x{i}"] = f.solve(2, rhs)
        out[f"xl{i}"] = f.solve(0, rhs)
        out[f"xu{i}"] = f.solve(1, rhs)
        out[f"var{i}"] = f.takahashi_diag()
        s = f.takahashi_full()
        out.update(mat(f"S{i}", s))
        parent, cpl = ref.symbolic(n, q.col_ptr, q.row_idx, perm)
        out[f"parent{i}"], out[f"cpl{i}"] = parent, cpl
    out["count"] = np.array(count)
    np.savez_compressed(os.path.join(HERE, name), **out)


def matern1d(ref):
    """C1: 1D Matérn regression, full size."""
    b = ref.build("matern1d", [999, 20.0, 2, 1.0, 100, 1001, 1e4, 0.01, 8, 2001, 1])
    out = {}
    for k in ["Q_prior", "A", "Q_post", "L"]:
        out.update(mat(k, b.mat(k)))
    for k in ["y", "noise", "points", "mean_post", "var_post", "z", "samples", "perm_amd"]:
        out[k] = b.vec(k)
    np.savez_compressed(os.path.join(HERE, "c1_matern1d.npz"), **out)


def matern2d(ref):
    """C2: 2D Matérn regression, full size (256² nodes, 2000
    observations, Rng(1002) interleaved (x, y) then noises), mean, Takahashi
    variances and the first 2 of the 16 samples (Rng(2002); z is re-drawn by the
    test through the Rng mirror). The factor L is not stored (8.1M entries)."""
    b = ref.build("matern2d", [255, 10.0, 2, 1.0, 2000, 1002, 400.0, 0.05, 2, 2002, 1])
    out = {}
    for k in ["A", "Q_post"]:
        out.update(mat(k, b.mat(k)))
    for k in ["y", "noise", "points", "mean_post", "var_post", "samples", "perm_amd"]:
        out[k] = b.vec(k)
    out["perm_amd"] = out["perm_amd"].astype(np.int32)
    np.savez_compressed(os.path.join(HERE, "c2_matern2d.npz"), **out)


def spatiotemporal(ref, kind, n_el, n_t, name, gn_iters=0):
    """C3 (heat) / C4 (Burgers) shapes at reduced size."""
    if kind == 0:
        p = [0, n_el, 0.0, 1.0, n_t, 1.0, 0.1, 0.0, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e6, 1003,
             0, 0, 1, 0]
    else:
        p = [1, n_el, -1.0, 1.0, n_t, 1.0, 0.01 / np.pi, 0.5, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e8,
             0, 1e12, gn_iters, 1, 1]
    b = ref.build("spatiotemporal", p)
    out = {"params": np.array(p, np.float64)}
    names = ["Q_prior", "S_prior", "A_ic", "Q_cond", "S_cond"]
    if kind == 1:
        names += ["Q_la", "J_at_mean_cond"]
    for k in names:
        out.update(mat(k, b.mat(k)))
    vecs = ["y_ic", "noise_ic", "mean_cond", "mean_post", "var_post"]
    if kind == 1:
        vecs += ["mode", "gn_objective", "gn_decrement", "gn_step", "gn_backtracks",
                 "f_at_mean_cond"]
    for k in vecs:
        out[k] = b.vec(k)
    np.savez_compressed(os.path.join(HERE, name), **out)


def allen_cahn(ref, n_cells, n_t, name, gn_iters=8):
    """C5 shape at reduced size: unit square, Allen-Cahn residual restated in
    oracle/ref_capi.cpp, driven by the reference gauss_newton / laplace_posterior
    / variance_takahashi (with a finite-difference check of its Jacobian)."""
    p = [n_cells, n_t, 0.5, 0.0025, 10, 1, 1, 10, 2, 1, 1.0, 1e6, 1005, 1e12, gn_iters, 1, 1, 1]
    b = ref.build("allen_cahn", p)
    out = {"params": np.array(p, np.float64), "fd_rel_err": np.array([b.scalar("fd_rel_err")])}
    for k in ["Q_prior", "Q_cond", "S_cond", "Q_la", "J_at_mean_cond"]:
        out.update(mat(k, b.mat(k)))
    for k in ["u0", "mean_cond", "f_at_mean_cond", "mode", "mean_post", "var_post",
              "gn_objective", "gn_decrement", "gn_step", "gn_backtracks"]:
        out[k] = b.vec(k)
    np.savez_compressed(os.path.join(HERE, name), **out)


def main():
    ref = Ref()
    if len(sys.argv) > 1:  # selected fixtures only, e.g. `make_golden.py matern2d`
        for name in sys.argv[1:]:
            globals()[name](ref)
        return
    corpus(ref, 50, 20240817, "corpus_acceptance.npz")   # acceptance.cpp:67 criterion 1
    corpus(ref, 12, 31415, "corpus_variance.npz")        # acceptance.cpp:652 criterion 10
    matern1d(ref)
    matern2d(ref)
    spatiotemporal(ref, 0, 19, 20, "c3_heat_20x20.npz")
    spatiotemporal(ref, 1, 19, 20, "c4_burgers_20x20.npz", gn_iters=4)
    allen_cahn(ref, 8, 16, "c5_allen_cahn_8x8x16.npz")
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
