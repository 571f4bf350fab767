"""Generates the BASELINE-size golden fixtures from the REFERENCE itself.

TEST INFRASTRUCTURE. Runs the unmodified reference (oracle/_ref/libgmrfref.so,
the /root/reference headers compiled by oracle/Makefile) single-threaded on the
seeded inputs of SURVEY §8(d), once, in the build container (hours for C4: the
reference's AMD factorization is ~190 s per GN step and its Takahashi pass
~3-4 h), and stores only the vectors the GPU tests compare against:

  c4_burgers_full.npz   C4 999 elements x 1000 slices (n = 1e6): 10-step GN
                        trace (objective, decrement, step, backtracks), mode,
                        Laplace Takahashi variances, reference stage timings.
  c3_heat_full.npz      C3 499 x 1000 (n = 500,000): IC-conditioned mean and
                        Takahashi variances, timings.
  c5_allen_cahn_<k>.npz C5 shape at k^2 nodes x (2k) slices (k = 16, 24, 32): 8-step
                        GN trace, mode, variances, timings (k = 32 is n = 65,536,
                        the largest the reference's int32 nnz(L) survives).
  c4_burgers_200.npz    C4 shape at 199 x 200 with the full 10-step GN budget.

Usage: python tests/golden/make_golden_full.py c4 | c3 | c5_16 | c5_24 | c5_32 | c4_200 | c4_500
       python tests/golden/make_golden_full.py floor:c4_200 ...
Each run writes its fixture atomically (tmp + rename) plus a .log with timings.

``order:<job>`` re-runs the unmodified reference chain with its fill-reducing
ordering (AMD in gauss_newton.hpp:139 and cholesky_factor, gmrf.hpp:55,160)
redirected to METIS nested dissection (oracle/_ref/libgmrfref_nd.so) and records
the move in floors.json under "<fixture>/order": the reference's ordering floor
(SURVEY §8(c) (i)), the primary tolerance scale of the GPU parity tests.

``floor_novar:<job>`` / ``order_novar:<job>`` are ``floor:`` / ``order:`` without the variance pass (the full-size C4
probe: the Takahashi pass alone is hours there).

``floor:<job>`` re-runs the same unmodified reference chain with every initial-
condition value multiplied by (1 ± 2⁻⁵²) (oracle/ref_capi.cpp ulp_perturb,
SURVEY §8(c) "floor2") and records in floors.json how far the reference's own
outputs move (GN objective / decrement, mode, variances, relative). That is the
reference's FP64 floor for the chain: one ulp of input noise, amplified by the
conditioning of H (Λ_pde = 1e12) and by the Gauss-Newton trajectory. GPU parity
is judged against a small multiple of it (tests/test_gpu_parity_full.py).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import REF_ND_SO, REF_SO, Ref  # noqa: E402

TIMERS = ["t_prior", "t_condition", "t_gn", "t_laplace_build", "t_variance"]


def _save(name, out, b, t_wall):
    times = {}
    for k in TIMERS:
        try:
            times[k] = float(b.scalar(k))
        except Exception:  # stage not run for this config
            pass
    times["t_wall"] = t_wall
    out["ref_times_json"] = np.array(json.dumps(times))
    tmp = os.path.join(HERE, name + ".tmp.npz")
    np.savez_compressed(tmp, **out)
    os.replace(tmp, os.path.join(HERE, name))
    print(name, json.dumps(times), flush=True)


FLOOR_SEED = 7
MODE = {"so": REF_SO, "tag": ""}  # order: jobs switch to the ND-ordering probe build


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _record_floor(name, b):
    """Compares a perturbed reference run with the committed fixture (waits for a
    fixture job started alongside to finish)."""
    for _ in range(6 * 240):
        if os.path.exists(os.path.join(HERE, name)):
            break
        time.sleep(10)
    z = np.load(os.path.join(HERE, name))
    f = {"seed": FLOOR_SEED} if MODE["tag"] == "/ulp" else {"ordering": "metis_nd"}
    for k, key in (("mean", "mode"), ("mean", "mean_post"), ("var", "var_post")):
        if key in z.files and k not in f:
            try:
                f[k] = _rel(b.vec(key), z[key])
            except Exception:  # stage not run by this probe (floor_novar)
                pass
    if "gn_objective" in z.files:
        for k in ("gn_objective", "gn_decrement"):
            v = b.vec(k)
            if len(v) == len(z[k]):
                d = np.abs(v - z[k]) / np.abs(z[k])
                f[k.replace("gn_", "")] = float(np.max(d))
                f[k.replace("gn_", "") + "_per_iter"] = [float(x) for x in d]
        f["same_trace"] = bool(np.array_equal(b.vec("gn_backtracks"), z["gn_backtracks"]))
    path = os.path.join(HERE, "floors.json")
    floors = json.load(open(path)) if os.path.exists(path) else {}
    floors[name + MODE["tag"]] = f
    with open(path + ".tmp", "w") as fh:
        json.dump(floors, fh, indent=1, sort_keys=True)
    os.replace(path + ".tmp", path)
    print("floor", name, f, flush=True)


def burgers(n_el, n_t, gn_iters, name, floor=False):
    # make_golden.spatiotemporal parameter layout (oracle/ref_capi.cpp:157-160)
    p = [1, n_el, -1.0, 1.0, n_t, 1.0, 0.01 / np.pi, 0.5, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e8,
         0, 1e12, gn_iters, 0 if MODE.get("novar") else 1, 1, 0,
         FLOOR_SEED if floor and MODE["tag"] == "/ulp" else 0]
    t0 = time.time()
    b = Ref(MODE["so"]).build("spatiotemporal", p)
    if floor:
        return _record_floor(name, b)
    out = {"params": np.array(p, np.float64)}
    keys = ["mean_cond", "mode", "mean_post", "var_post", "gn_objective", "gn_decrement",
            "gn_step", "gn_backtracks"]
    if n_el * n_t > 500000:  # full size: the Laplace mean is the mode; keep the fixture small
        keys = [k for k in keys if k not in ("mean_cond", "mean_post")]
    for k in keys:
        out[k] = b.vec(k)
    out["gn_converged"] = np.array(b.scalar("gn_converged"))
    _save(name, out, b, time.time() - t0)


def heat(n_el, n_t, name, floor=False):
    p = [0, n_el, 0.0, 1.0, n_t, 1.0, 0.1, 0.0, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e6, 1003,
         0, 0, 1, 0, 0, FLOOR_SEED if floor and MODE["tag"] == "/ulp" else 0]
    t0 = time.time()
    b = Ref(MODE["so"]).build("spatiotemporal", p)
    if floor:
        return _record_floor(name, b)
    out = {"params": np.array(p, np.float64)}
    for k in ["y_ic", "mean_post", "var_post"]:
        out[k] = b.vec(k)
    _save(name, out, b, time.time() - t0)


def allen_cahn(n_cells, n_t, name, gn_iters=8, floor=False):
    p = [n_cells, n_t, 0.5, 0.0025, 10, 1, 1, 10, 2, 1, 1.0, 1e6, 1005, 1e12, gn_iters, 1, 1, 1,
         FLOOR_SEED if floor and MODE["tag"] == "/ulp" else 0]
    t0 = time.time()
    b = Ref(MODE["so"]).build("allen_cahn", p)
    if floor:
        return _record_floor(name, b)
    out = {"params": np.array(p, np.float64), "fd_rel_err": np.array([b.scalar("fd_rel_err")])}
    for k in ["u0", "mean_cond", "mode", "mean_post", "var_post", "gn_objective",
              "gn_decrement", "gn_step", "gn_backtracks"]:
        out[k] = b.vec(k)
    out["gn_converged"] = np.array(b.scalar("gn_converged"))
    _save(name, out, b, time.time() - t0)


def matern(dim, name, floor=False):
    """C1 / C2 regression (make_golden.matern1d / matern2d parameters); floor runs
    only (the full fixtures are make_golden.py's)."""
    p = ([999, 20.0, 2, 1.0, 100, 1001, 1e4, 0.01, 8, 2001, 1] if dim == 1 else
         [255, 10.0, 2, 1.0, 2000, 1002, 400.0, 0.05, 2, 2002, 1])
    assert floor and MODE["tag"] == "/order", "regression fixtures come from make_golden.py"
    b = Ref(MODE["so"]).build("matern1d" if dim == 1 else "matern2d", p)
    return _record_floor(name, b)


JOBS = {
    "c1": lambda fl: matern(1, "c1_matern1d.npz", fl),
    "c2": lambda fl: matern(2, "c2_matern2d.npz", fl),
    "c4": lambda fl: burgers(999, 1000, 10, "c4_burgers_full.npz", fl),
    "c4_200": lambda fl: burgers(199, 200, 10, "c4_burgers_200.npz", fl),
    "c4_500": lambda fl: burgers(499, 500, 10, "c4_burgers_500.npz", fl),
    "c3": lambda fl: heat(499, 1000, "c3_heat_full.npz", fl),
    "c5_16": lambda fl: allen_cahn(15, 32, "c5_allen_cahn_16.npz", floor=fl),
    "c5_24": lambda fl: allen_cahn(23, 48, "c5_allen_cahn_24.npz", floor=fl),
    "c5_32": lambda fl: allen_cahn(31, 64, "c5_allen_cahn_32.npz", floor=fl),
}

if __name__ == "__main__":
    for job in sys.argv[1:]:
        kind = job.split(":")[0] if ":" in job else ""
        if kind == "order":
            MODE.update(so=REF_ND_SO, tag="/order")
        elif kind == "floor":
            MODE.update(tag="/ulp")
        elif kind == "order_novar":
            MODE.update(so=REF_ND_SO, tag="/order", novar=True)
        elif kind == "floor_novar":
            # full-size probe without the Takahashi pass (hours at n = 1e6): GN trace
            # and mode floors only
            MODE.update(tag="/ulp", novar=True)
        JOBS[job.split(":")[-1]](kind != "")
