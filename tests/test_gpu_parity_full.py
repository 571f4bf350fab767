"""GPU parity at BASELINE sizes against the reference run on the same seeded
inputs (fixtures from tests/golden/make_golden_full.py: the unmodified
reference, single-threaded, hours for C4).

Every fixture is the reference's own chain (spatiotemporal_prior → condition_on
→ gauss_newton → laplace_posterior → variance_takahashi, AMD ordering); the
product runs its own chain (device assembly, ND-ordered supernodal factor) from
the same inputs. Required (north_star):
  * identical GN iteration counts, backtracks and step sizes (exact);
  * mean (mode), marginal variances, GN objectives and decrements within the
    north_star bound (mean 1e-10, variances 1e-8) or, where the reference's
    own FP64 floor is above it, within K = 10 times that floor (SURVEY §8(c)
    (i), k ≈ 2-10).
The floor (tests/golden/floors.json, committed next to the fixtures) is the
larger of two self-consistency probes of the UNMODIFIED reference on the same
inputs (tests/golden/make_golden_full.py): its chain with the AMD ordering
replaced by METIS nested dissection ("/order"), and its chain with every input
value perturbed by one ulp ("/ulp"). The space-time systems are
ill-conditioned (Λ_pde = 1e12, slack ε = 1e-10) and 10 Gauss-Newton steps
amplify rounding, so these floors reach 1e-8..1e-4; the product's measured
errors and their ratio to the floor are printed (and appended to
$GMRF_PARITY_REPORT) for the record.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior
from test_gpu_spacetime import rel, spec_ac, spec_from

pytestmark = pytest.mark.gpu

REPORT = os.environ.get("GMRF_PARITY_REPORT")  # optional JSON-lines sink for the measured errors


def _load(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated (tests/golden/make_golden_full.py)")
    return np.load(path)


def _report(name, **kw):
    print(name, kw)
    if REPORT:
        with open(REPORT, "a") as f:
            f.write(json.dumps({"fixture": name, **kw}) + "\n")


def _check_trace(z, trace):
    assert len(trace) == len(z["gn_objective"])  # identical GN iteration count
    np.testing.assert_array_equal([t.backtracks for t in trace], z["gn_backtracks"])
    np.testing.assert_array_equal([t.step_size for t in trace], z["gn_step"])
    obj = np.array([t.objective for t in trace])
    dec = np.array([t.decrement for t in trace])
    # a decrement below the reference's own convergence resolution (it stops at
    # 0.5·dec² <= 1e-14·(1 + |objective|), gauss_newton.hpp:187-188) is compared on
    # that scale: relative error of a quantity the reference treats as zero means nothing
    res = np.sqrt(2e-14 * (1.0 + np.abs(z["gn_objective"])))
    return (float(np.max(np.abs(obj - z["gn_objective"]) / np.abs(z["gn_objective"]))),
            float(np.max(np.abs(dec - z["gn_decrement"]) / np.maximum(np.abs(z["gn_decrement"]), res))))


K = 10.0
BOUND = {"mean": 1e-10, "var": 1e-8, "objective": 1e-12, "decrement": 1e-12}


def _floors(name):
    path = os.path.join(GOLDEN, "floors.json")
    fl = json.load(open(path)) if os.path.exists(path) else {}
    probes = [fl[k] for k in (name + "/order", name + "/ulp") if k in fl]
    if name + "/order" not in fl:
        # the product factors in a nested-dissection order, the fixture's reference run
        # in AMD order: the ordering probe is the tolerance scale that applies
        pytest.skip(f"ordering floor for {name} not measured yet (make_golden_full.py order:)")
    out = {k: max(p.get(k, 0.0) for p in probes) for k in BOUND}
    if not any("var" in p for p in probes):
        # full-size probes skip the reference's Takahashi pass (hours at n = 1e6;
        # make_golden_full.py order_novar: / floor_novar:): the variance floor is the
        # measured mean floor times the SMALLEST var/mean floor ratio the same family
        # shows at the sizes where both were measured (0.5-0.8 for config 4)
        fam = name.split("_")[0]
        ratios = [v["var"] / v["mean"] for key, v in fl.items()
                  if key.startswith(fam) and "var" in v and v.get("mean", 0.0) > 0.0]
        out["var"] = out["mean"] * min(ratios)
    return out


def _judge(name, errs):
    fl = _floors(name)
    tol = {k: max(BOUND[k], K * fl[k]) for k in errs}
    _report(name, **{k: errs[k] for k in errs}, **{"floor_" + k: fl[k] for k in errs},
            **{"ratio_" + k: errs[k] / max(fl[k], 1e-300) for k in errs})
    bad = {k: (errs[k], tol[k]) for k in errs if not errs[k] <= tol[k]}
    assert not bad, bad


BURGERS = ["c4_burgers_200.npz", "c4_burgers_500.npz", "c4_burgers_full.npz"]
ALLEN_CAHN = ["c5_allen_cahn_16.npz", "c5_allen_cahn_24.npz", "c5_allen_cahn_32.npz"]


@pytest.mark.parametrize("fixture", BURGERS)
def test_burgers_posterior_matches_reference(fixture):
    z = _load(fixture)
    p = z["params"]
    post = SpaceTimePosterior(spec_from(p), GaussNewtonConfig(max_iters=int(p[19])))
    x = post.spec.node_x()
    u0 = -np.sin(np.pi * x)
    mean, var, trace, conv = post.run(u0, variances=True)
    eobj, edec = _check_trace(z, trace)
    _judge(fixture, {"objective": eobj, "decrement": edec, "mean": rel(mean, z["mode"]),
                     "var": rel(var, z["var_post"])})


def test_heat_full_matches_reference():
    z = _load("c3_heat_full.npz")
    p = z["params"]
    post = SpaceTimePosterior(spec_from(p))
    mean, var, trace, conv = post.run(z["y_ic"], variances=True)
    _judge("c3_heat_full.npz", {"mean": rel(mean, z["mean_post"]), "var": rel(var, z["var_post"])})


@pytest.mark.parametrize("fixture", ALLEN_CAHN)
def test_allen_cahn_posterior_matches_reference(fixture):
    z = _load(fixture)
    p = z["params"]
    post = SpaceTimePosterior(spec_ac(p), GaussNewtonConfig(max_iters=int(p[14])))
    mean, var, trace, conv = post.run(z["u0"], variances=True)
    eobj, edec = _check_trace(z, trace)
    _judge(fixture, {"objective": eobj, "decrement": edec, "mean": rel(mean, z["mode"]),
                     "var": rel(var, z["var_post"])})
