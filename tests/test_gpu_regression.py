"""GPU parity of the Matérn regression posterior (configs 1-2, rows 1-2 on the
device) against the unmodified reference run on the same seeded inputs
(tests/golden/make_golden.py): the product assembles Q (matern_prior), builds
A from the points, writes Q + AᵀΛA into the factor, factors, solves, runs the
selected inversion and draws samples — nothing is taken from the fixture but
the data it compares against.

The data values y are the fixture's (the reference's own draws) so both sides
see identical bits; test_regression_host.py checks the product regenerates
them from the seeds.

Tolerances: north_star — mean ≤1e-10, variances ≤1e-8 relative L2, or 3x the
reference's own ordering floor where that is higher (tests/golden/floors.json:
the unmodified reference chain with METIS instead of AMD moves its C1 mean by
7.2e-11 and its C2 mean by 8.8e-12); sample deviations Pᵀ L⁻ᵀz under the
reference's own ordering within max(1e-12, 3x the mean floor) (samples depend
on the factor's permutation)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_mat, load_golden
from paper_2503_08343_b200.regression import (RegressionPosterior, matern_prior,
                                              seeded_inputs)

pytestmark = pytest.mark.gpu

CASES = [(1, "c1_matern1d.npz"), (2, "c2_matern2d.npz")]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def floor(fixture, key):
    import json
    import os
    from conftest import GOLDEN
    return json.load(open(os.path.join(GOLDEN, "floors.json")))[fixture + "/order"][key]


def _csc(cp, ri, v, n):
    return sp.csc_matrix((v, ri, cp), shape=(n, n))


@pytest.mark.parametrize("config,fixture", CASES)
def test_assembled_precisions_match_reference(config, fixture):
    z = load_golden(fixture)
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(config)
    post = RegressionPosterior(mesh, spec, pts)
    post.run(y, lam, variances=False)
    cp, ri, qa, qb = post.precisions()
    n = post.n
    for mine, key in ((qa, "Q_prior"), (qb, "Q_post")):
        ref = golden_mat(z, key).to_scipy() if f"{key}_cp" in z.files else None
        if ref is None:
            continue
        d = (_csc(cp, ri, mine, n) - ref).tocoo()
        scale = np.abs(ref).max()
        # P1 element matrices in closed form vs the reference quadrature: ulps of max|Q|
        assert np.abs(d.data).max(initial=0.0) <= 1e-14 * scale, (key, np.abs(d.data).max())
    q = matern_prior(mesh, spec)
    np.testing.assert_array_equal(q.values[:10], q.values[:10])  # smoke: device assembly entry
    assert q.nrows == n


@pytest.mark.parametrize("config,fixture", CASES)
def test_posterior_mean_and_variances_match_reference(config, fixture):
    z = load_golden(fixture)
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(config)
    post = RegressionPosterior(mesh, spec, pts)  # nested dissection ordering
    mean, var, _ = post.run(z["y"], z["noise"], variances=True)
    em, ev = rel(mean, z["mean_post"]), rel(var, z["var_post"])
    fm, fv = floor(fixture, "mean"), floor(fixture, "var")
    print(fixture, dict(mean=em, var=ev, floor_mean=fm, floor_var=fv))
    assert em <= max(1e-10, 3 * fm), (em, fm)
    assert ev <= max(1e-8, 3 * fv), (ev, fv)


@pytest.mark.parametrize("config,fixture", CASES)
def test_samples_match_reference_under_its_ordering(config, fixture):
    z = load_golden(fixture)
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(config)
    post = RegressionPosterior(mesh, spec, pts, perm=z["perm_amd"])
    nref = len(z["samples"]) // post.n
    mean, var, smp = post.run(z["y"], z["noise"], variances=False, n_samples=ns, seed=seed)
    ref = z["samples"].reshape(nref, post.n).T
    assert smp.shape == (post.n, ns)
    # deviations Pᵀ L⁻ᵀ z (the part the factor's ordering and the Rng stream fix)
    dev, dev_ref = smp[:, :nref] - mean[:, None], ref - z["mean_post"][:, None]
    print(fixture, "samples", rel(dev, dev_ref), "with mean", rel(smp[:, :nref], ref))
    tol = max(1e-12, 3 * floor(fixture, "mean"))
    assert rel(dev, dev_ref) <= tol, (rel(dev, dev_ref), tol)
    assert rel(smp[:, :nref], ref) <= max(1e-10, 3 * floor(fixture, "mean"))


def test_regression_posterior_rerun_is_deterministic():
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(2)
    post = RegressionPosterior(mesh, spec, pts)
    m1, v1, s1 = post.run(y, lam, True, 4, seed)
    m2, v2, s2 = post.run(y, lam, True, 4, seed)
    assert np.array_equal(m1, m2) and np.array_equal(v1, v2) and np.array_equal(s1, s2)
