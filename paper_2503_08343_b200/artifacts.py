"""Experiment artifacts in the reference's on-disk formats.

Mirrors ``detail::write_artifacts`` (bench/runner.hpp:674-722) so downstream
tooling written against the reference reads these files unchanged:

* ``result.json`` — ordered keys kind, resolution, order, n_dofs, seed,
  relative_l2_error_percent, phases{prior_construction_s, conditioning_solve_s,
  variance_s, sampling_s, total_s}, gauss_newton{iterations, final_decrement,
  converged}, optional fem_baseline{time_s, error_percent}; 2-space indent
  (nlohmann ``dump(2)``); a NaN error (no reference truth) is written as null,
  as nlohmann does;
* ``solution.csv`` — ``x,mean,stddev`` (1-D), ``t,x,mean,stddev`` (space-time
  Burgers kinds), else ``x,y,mean,stddev``; every real as ``%.9g``
  (runner.hpp:88-92), stddev left empty when no variances were computed;
* ``trace.csv`` — ``iteration,objective,decrement,step_size,backtracks,
  cg_iterations`` (written only when there is a Gauss-Newton trace).

``spacetime_artifacts`` fills them from a :class:`SpaceTimePosterior` run the
way ``run_burgers`` does (runner.hpp:655-669: coordinates (t, x) per DoF in
slice-major order, stddev = sqrt(variance)). The 2-D space-time case (config 5,
no reference counterpart) writes ``t,x,y,mean,stddev``.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np


def format_real(v: float) -> str:
    """runner.hpp:88-92: snprintf("%.9g")."""
    return "%.9g" % float(v)


@dataclass
class Phases:
    """ResultRecord::phases (runner.hpp:683-687); total = the sum."""
    prior_construction_s: float = 0.0
    conditioning_solve_s: float = 0.0
    variance_s: float = 0.0
    sampling_s: float = 0.0

    def total(self) -> float:
        return (self.prior_construction_s + self.conditioning_solve_s + self.variance_s +
                self.sampling_s)


@dataclass
class ResultRecord:
    kind: str
    resolution: int
    order: int
    n_dofs: int
    seed: int
    relative_l2_error_percent: float = math.nan
    phases: Phases = field(default_factory=Phases)
    gn_iterations: int = 0
    gn_final_decrement: float = 0.0
    gn_converged: bool = False
    fem_baseline_time_s: float = -1.0
    fem_baseline_error_percent: float = math.nan


def _num(v):
    return None if isinstance(v, float) and not math.isfinite(v) else v


def write_artifacts(output_dir: str, rec: ResultRecord, coords: np.ndarray, coord_dim: int,
                    mean: np.ndarray, stddev: np.ndarray | None, trace=()) -> None:
    """runner.hpp:674-722. ``coords`` is (n, coord_dim) or flat, DoF-major."""
    os.makedirs(output_dir, exist_ok=True)
    j = {
        "kind": rec.kind,
        "resolution": int(rec.resolution),
        "order": int(rec.order),
        "n_dofs": int(rec.n_dofs),
        "seed": int(rec.seed),
        "relative_l2_error_percent": _num(float(rec.relative_l2_error_percent)),
        "phases": {
            "prior_construction_s": rec.phases.prior_construction_s,
            "conditioning_solve_s": rec.phases.conditioning_solve_s,
            "variance_s": rec.phases.variance_s,
            "sampling_s": rec.phases.sampling_s,
            "total_s": rec.phases.total(),
        },
        "gauss_newton": {
            "iterations": int(rec.gn_iterations),
            "final_decrement": _num(float(rec.gn_final_decrement)),
            "converged": bool(rec.gn_converged),
        },
    }
    if rec.fem_baseline_time_s >= 0.0:
        j["fem_baseline"] = {"time_s": rec.fem_baseline_time_s,
                             "error_percent": _num(float(rec.fem_baseline_error_percent))}
    with open(os.path.join(output_dir, "result.json"), "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")

    coords = np.asarray(coords, np.float64).reshape(len(mean), coord_dim)
    if coord_dim == 1:
        head = "x,mean,stddev"
    elif coord_dim == 3:
        head = "t,x,y,mean,stddev"
    elif rec.kind in ("burgers_li", "burgers_cole_hopf"):
        head = "t,x,mean,stddev"
    else:
        head = "x,y,mean,stddev"
    lines = [head]
    for i in range(len(mean)):
        cs = ",".join(format_real(c) for c in coords[i])
        sd = "" if stddev is None else format_real(stddev[i])
        lines.append("%s,%s,%s" % (cs, format_real(mean[i]), sd))
    with open(os.path.join(output_dir, "solution.csv"), "w") as f:
        f.write("\n".join(lines) + "\n")

    if len(trace):
        rows = ["iteration,objective,decrement,step_size,backtracks,cg_iterations"]
        for t in trace:
            rows.append("%d,%s,%s,%s,%d,%d" % (t.iter, format_real(t.objective),
                                               format_real(t.decrement), format_real(t.step_size),
                                               t.backtracks, getattr(t, "cg_iterations", 0)))
        with open(os.path.join(output_dir, "trace.csv"), "w") as f:
            f.write("\n".join(rows) + "\n")


def spacetime_coords(spec, n_space: int) -> tuple[np.ndarray, int]:
    """(t, x) or (t, x, y) per joint DoF t·n_s + d (runner.hpp:663-667)."""
    t_grid = np.linspace(0.0, spec.t_end, spec.n_t)
    if getattr(spec, "dim", 1) == 2:
        xy = spec.node_xy()
        t = np.repeat(t_grid, n_space)
        return np.stack([t, np.tile(xy[:, 0], spec.n_t), np.tile(xy[:, 1], spec.n_t)], axis=1), 3
    x = spec.node_x()
    return np.stack([np.repeat(t_grid, n_space), np.tile(x, spec.n_t)], axis=1), 2


def spacetime_artifacts(output_dir: str, post, spec, mean, var, trace, converged, seed: int = 0,
                        kind: str | None = None) -> ResultRecord:
    """Artifacts of one SpaceTimePosterior.run (the run_burgers record fields)."""
    if kind is None:
        kind = "allen_cahn" if getattr(spec, "residual", 1) == 2 else "burgers_li"
    info = post.info()
    n_space = int(info.n_space)
    rec = ResultRecord(kind=kind, resolution=int(spec.n_el), order=1, n_dofs=int(info.n), seed=seed)
    rec.phases = Phases(
        prior_construction_s=(info.setup_host_ms + info.assemble_ms) * 1e-3,
        conditioning_solve_s=(info.condition_ms + info.gn_ms + info.laplace_ms) * 1e-3,
        variance_s=info.selinv_ms * 1e-3)
    rec.gn_iterations = len(trace)
    rec.gn_final_decrement = trace[-1].decrement if trace else 0.0
    rec.gn_converged = bool(converged)
    coords, cd = spacetime_coords(spec, n_space)
    sd = None if var is None else np.sqrt(np.maximum(var, 0.0))
    write_artifacts(output_dir, rec, coords, cd, mean, sd, trace)
    return rec
