"""Artifact formats (result.json / solution.csv / trace.csv) against the
reference writer's rules (bench/runner.hpp:674-722, format_real :88-92)."""
import json
import math
import os
from collections import namedtuple

import numpy as np
import pytest

from paper_2503_08343_b200 import artifacts as A

It = namedtuple("It", "iter objective decrement step_size backtracks")


def test_format_real_matches_snprintf_9g():
    assert A.format_real(0.1) == "0.1"
    assert A.format_real(1.0 / 3.0) == "0.333333333"
    assert A.format_real(-2.5e-7) == "-2.5e-07"
    assert A.format_real(123456789012.0) == "1.23456789e+11"
    assert A.format_real(0.0) == "0"


def test_write_artifacts_layout(tmp_path):
    rec = A.ResultRecord(kind="burgers_li", resolution=4, order=1, n_dofs=6, seed=7)
    rec.phases = A.Phases(0.5, 1.25, 0.25, 0.0)
    rec.gn_iterations, rec.gn_final_decrement, rec.gn_converged = 2, 3.5e-3, False
    coords = np.array([[0.0, -1.0], [0.0, 1.0], [0.5, -1.0], [0.5, 1.0], [1.0, -1.0], [1.0, 1.0]])
    mean = np.arange(6) / 7.0
    sd = np.full(6, 0.25)
    trace = [It(1, 10.0, 2.0, 0.5, 1), It(2, 1.0 / 3.0, 3.5e-3, 1.0, 0)]
    A.write_artifacts(str(tmp_path), rec, coords, 2, mean, sd, trace)
    txt = open(tmp_path / "result.json").read()
    j = json.loads(txt)
    assert list(j) == ["kind", "resolution", "order", "n_dofs", "seed", "relative_l2_error_percent",
                       "phases", "gauss_newton"]
    assert j["relative_l2_error_percent"] is None  # NaN → null, as nlohmann writes it
    assert list(j["phases"]) == ["prior_construction_s", "conditioning_solve_s", "variance_s",
                                 "sampling_s", "total_s"]
    assert j["phases"]["total_s"] == pytest.approx(2.0)
    assert j["gauss_newton"] == {"iterations": 2, "final_decrement": 3.5e-3, "converged": False}
    assert txt.startswith('{\n  "kind": "burgers_li",\n')
    sol = open(tmp_path / "solution.csv").read().splitlines()
    assert sol[0] == "t,x,mean,stddev"
    assert sol[2] == "0,1,0.142857143,0.25"
    tr = open(tmp_path / "trace.csv").read().splitlines()
    assert tr == ["iteration,objective,decrement,step_size,backtracks,cg_iterations",
                  "1,10,2,0.5,1,0", "2,0.333333333,0.0035,1,0,0"]


def test_write_artifacts_variants(tmp_path):
    rec = A.ResultRecord(kind="poisson", resolution=2, order=1, n_dofs=3, seed=0,
                         relative_l2_error_percent=1.5, fem_baseline_time_s=0.1,
                         fem_baseline_error_percent=2.0)
    A.write_artifacts(str(tmp_path / "a"), rec, np.array([0.0, 0.5, 1.0]), 1, np.ones(3), None)
    sol = open(tmp_path / "a" / "solution.csv").read().splitlines()
    assert sol == ["x,mean,stddev", "0,1,", "0.5,1,", "1,1,"]
    assert not os.path.exists(tmp_path / "a" / "trace.csv")
    j = json.load(open(tmp_path / "a" / "result.json"))
    assert j["fem_baseline"] == {"time_s": 0.1, "error_percent": 2.0}
    rec.kind = "darcy"
    A.write_artifacts(str(tmp_path / "b"), rec, np.zeros((3, 2)), 2, np.ones(3), np.ones(3))
    assert open(tmp_path / "b" / "solution.csv").readline().strip() == "x,y,mean,stddev"


def test_spacetime_coords_order():
    from paper_2503_08343_b200.spacetime import SpaceTimeSpec
    sp1 = SpaceTimeSpec.burgers(n_el=3, n_t=2)
    c, d = A.spacetime_coords(sp1, 4)
    assert d == 2 and c.shape == (8, 2)
    np.testing.assert_allclose(c[:4, 0], 0.0)
    np.testing.assert_allclose(c[4:, 0], 1.0)
    np.testing.assert_allclose(c[:4, 1], sp1.node_x())
    sp2 = SpaceTimeSpec.allen_cahn(n_cells=2, n_t=3)
    c, d = A.spacetime_coords(sp2, 9)
    assert d == 3 and c.shape == (27, 3)
    np.testing.assert_allclose(c[9:18, 0], 0.25)
    np.testing.assert_allclose(c[:9, 1:], sp2.node_xy())
    assert math.isclose(c[-1, 0], 0.5)


@pytest.mark.gpu
def test_spacetime_run_artifacts(tmp_path):
    from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec
    spec = SpaceTimeSpec.burgers(n_el=39, n_t=40)
    post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=3))
    mean, var, trace, conv = post.run(-np.sin(np.pi * spec.node_x()))
    rec = A.spacetime_artifacts(str(tmp_path), post, spec, mean, var, trace, conv, seed=1004)
    assert rec.n_dofs == 40 * 40
    sol = open(tmp_path / "solution.csv").read().splitlines()
    assert sol[0] == "t,x,mean,stddev" and len(sol) == 1 + 40 * 40
    last = sol[-1].split(",")
    assert float(last[0]) == pytest.approx(1.0) and float(last[1]) == pytest.approx(1.0)
    assert float(last[2]) == pytest.approx(mean[-1], rel=1e-8, abs=1e-12)
    assert float(last[3]) == pytest.approx(math.sqrt(var[-1]), rel=1e-8)
    tr = open(tmp_path / "trace.csv").read().splitlines()
    assert len(tr) == 1 + len(trace)
    j = json.load(open(tmp_path / "result.json"))
    assert j["gauss_newton"]["iterations"] == len(trace)
    assert j["phases"]["variance_s"] > 0.0
