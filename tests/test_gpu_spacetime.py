"""GPU parity of the space-time pipeline (rows 1-2 and the GN-Laplace chain)
against the reference (golden fixtures from tests/golden/make_golden.py).

Function evaluations (assembled Q_cond, q_eff = sym(S Sᵀ), the Burgers
residual and Jacobian) are compared tightly. Solutions of the space-time
systems are compared against the reference's own FP64 floor measured in the
same test with the C restatement (the reference's mean moves by
~1e-5 when only the ordering changes on these matrices).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_mat, load_golden
from paper_2503_08343_b200.spacetime import MaternSpec, SpaceTimePosterior, SpaceTimeSpec

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def spec_from(params):
    p = params
    return SpaceTimeSpec(n_el=int(p[1]), xa=p[2], xb=p[3], n_t=int(p[4]), t_end=p[5],
                         diffusion=p[6], advection=p[7],
                         noise=MaternSpec(p[8], int(p[9]), p[10]),
                         init=MaternSpec(p[11], int(p[12]), p[13]), tau=p[14], eps=p[15],
                         dirichlet=True, ic_noise_prec=p[16], residual=int(p[0]),
                         pde_noise_prec=p[18])


def ours_matrix(post, which):
    cp, ri, qc, qe = post.pattern()
    v = qc if which == "cond" else qe
    return sp.csc_matrix((v, ri, cp), shape=(post.n, post.n))


def ordering_floor(port, q, b):
    """‖x(natural) − x(reverse)‖/‖x‖ of the reference algorithm on the same Q bits."""
    n = q.shape[0]
    q = q.tocsc()
    q.sort_indices()
    xs = []
    for perm in (np.arange(n), np.arange(n)[::-1].copy()):
        lcp, lri, lv, bad = port.cholesky(n, q.indptr, q.indices, q.data, perm)
        assert bad == -1
        xs.append(port.solve(n, lcp, lri, lv, perm, 2, b)[:, 0])
    return rel(xs[0], xs[1]), xs[0]


@pytest.mark.parametrize("fixture", ["c3_heat_20x20.npz", "c4_burgers_20x20.npz"])
def test_assembled_precisions_match_reference(fixture):
    z = load_golden(fixture)
    post = SpaceTimePosterior(spec_from(z["params"]))
    qref = golden_mat(z, "Q_cond").to_scipy()
    q = ours_matrix(post, "cond")
    assert sp.linalg.norm(q - qref) / sp.linalg.norm(qref) <= 1e-13
    s = golden_mat(z, "S_cond").to_scipy()
    qeff_ref = (s @ s.T)
    qeff_ref = 0.5 * (qeff_ref + qeff_ref.T)
    qe = ours_matrix(post, "eff")
    assert sp.linalg.norm(qe - qeff_ref) / sp.linalg.norm(qeff_ref) <= 1e-13


def test_burgers_residual_and_jacobian_match_reference():
    z = load_golden("c4_burgers_20x20.npz")
    post = SpaceTimePosterior(spec_from(z["params"]))
    u = z["mean_cond"]
    f = post.residual(u)
    assert rel(f, z["f_at_mean_cond"]) <= 1e-12
    rp, ci, v = post.jacobian(u)
    j = sp.csr_matrix((v, ci, rp), shape=(len(f), post.n))
    jref = golden_mat(z, "J_at_mean_cond").to_scipy()
    assert sp.linalg.norm(j - jref) / sp.linalg.norm(jref) <= 1e-13
    # same structural pattern (the reference keeps the θ=1 zero block too)
    assert (j != 0).sum() <= jref.nnz and j.nnz == jref.nnz


def test_heat_posterior_vs_reference(port):
    z = load_golden("c3_heat_20x20.npz")
    post = SpaceTimePosterior(spec_from(z["params"]))
    mean, var, trace, conv = post.run(z["y_ic"], variances=True)
    assert trace == []
    qref = golden_mat(z, "Q_cond").to_scipy()
    a = golden_mat(z, "A_ic").to_scipy()
    rhs = a.T @ (z["noise_ic"] * z["y_ic"])
    floor, _ = ordering_floor(port, qref, rhs)
    assert rel(mean, z["mean_post"]) <= max(10 * floor, 1e-10), (rel(mean, z["mean_post"]), floor)
    assert rel(var, z["var_post"]) <= 1e-8


def test_burgers_gn_laplace_vs_reference(port):
    z = load_golden("c4_burgers_20x20.npz")
    p = z["params"]
    from paper_2503_08343_b200.spacetime import GaussNewtonConfig
    post = SpaceTimePosterior(spec_from(p), GaussNewtonConfig(max_iters=int(p[19])))
    mean, var, trace, conv = post.run(z["y_ic"], variances=True)
    assert len(trace) == len(z["gn_objective"])            # identical GN iteration count
    np.testing.assert_array_equal([t.backtracks for t in trace], z["gn_backtracks"])
    np.testing.assert_array_equal([t.step_size for t in trace], z["gn_step"])
    obj = np.array([t.objective for t in trace])
    dec = np.array([t.decrement for t in trace])
    assert np.max(np.abs(obj - z["gn_objective"]) / np.abs(z["gn_objective"])) <= 1e-8
    assert np.max(np.abs(dec - z["gn_decrement"]) / np.abs(z["gn_decrement"])) <= 1e-6
    qla = golden_mat(z, "Q_la").to_scipy()
    floor, _ = ordering_floor(port, qla, qla @ z["mode"])
    assert rel(mean, z["mode"]) <= max(10 * floor, 1e-10), (rel(mean, z["mode"]), floor)
    assert rel(var, z["var_post"]) <= 1e-8


# ---- config 5 shape: 2-D unit square, Allen-Cahn residual -------------------
def spec_ac(params):
    p = params
    return SpaceTimeSpec(n_el=int(p[0]), xa=0.0, xb=1.0, n_t=int(p[1]), t_end=p[2], diffusion=p[3],
                         advection=0.0, noise=MaternSpec(p[4], int(p[5]), p[6]),
                         init=MaternSpec(p[7], int(p[8]), p[9]), tau=p[10], dirichlet=False,
                         ic_noise_prec=p[11], residual=2, pde_noise_prec=p[13], dim=2)


def test_allen_cahn_assembly_residual_jacobian_match_reference():
    z = load_golden("c5_allen_cahn_8x8x16.npz")
    post = SpaceTimePosterior(spec_ac(z["params"]))
    assert post.n == 81 * 16
    qref = golden_mat(z, "Q_cond").to_scipy()
    q = ours_matrix(post, "cond")
    assert sp.linalg.norm(q - qref) / sp.linalg.norm(qref) <= 1e-13
    s = golden_mat(z, "S_cond").to_scipy()
    qeff_ref = s @ s.T
    qeff_ref = 0.5 * (qeff_ref + qeff_ref.T)
    assert sp.linalg.norm(ours_matrix(post, "eff") - qeff_ref) / sp.linalg.norm(qeff_ref) <= 1e-13
    u = z["mean_cond"]
    f = post.residual(u)
    assert rel(f, z["f_at_mean_cond"]) <= 1e-12
    rp, ci, v = post.jacobian(u)
    j = sp.csr_matrix((v, ci, rp), shape=(len(f), post.n))
    jref = golden_mat(z, "J_at_mean_cond").to_scipy()
    assert sp.linalg.norm(j - jref) / sp.linalg.norm(jref) <= 1e-13
    assert j.nnz == jref.nnz


def test_allen_cahn_gn_laplace_vs_reference(port):
    z = load_golden("c5_allen_cahn_8x8x16.npz")
    p = z["params"]
    from paper_2503_08343_b200.spacetime import GaussNewtonConfig
    post = SpaceTimePosterior(spec_ac(p), GaussNewtonConfig(max_iters=int(p[14])))
    mean, var, trace, conv = post.run(z["u0"], variances=True)
    assert len(trace) == len(z["gn_objective"])            # identical GN iteration count
    np.testing.assert_array_equal([t.backtracks for t in trace], z["gn_backtracks"])
    np.testing.assert_array_equal([t.step_size for t in trace], z["gn_step"])
    obj = np.array([t.objective for t in trace])
    assert np.max(np.abs(obj - z["gn_objective"]) / np.abs(z["gn_objective"])) <= 1e-8
    qla = golden_mat(z, "Q_la").to_scipy()
    floor, _ = ordering_floor(port, qla, qla @ z["mode"])
    assert rel(mean, z["mode"]) <= max(10 * floor, 1e-10), (rel(mean, z["mode"]), floor)
    assert rel(var, z["var_post"]) <= 1e-8


def test_gn_stagnation_carries_trace():
    """GaussNewtonStagnation(msg, trace) (gauss_newton.hpp:208-214): with no
    backtracks allowed, the reference's first C4 step (step 0.25 at 20x20) fails
    the Armijo test; the exception carries the trace up to that iteration."""
    from paper_2503_08343_b200.spacetime import GaussNewtonConfig, GaussNewtonStagnation
    z = load_golden("c4_burgers_20x20.npz")
    p = z["params"]
    assert z["gn_backtracks"][0] > 0
    post = SpaceTimePosterior(spec_from(p), GaussNewtonConfig(max_iters=4, max_backtracks=0))
    with pytest.raises(GaussNewtonStagnation) as ei:
        post.run(z["y_ic"], variances=False)
    tr = ei.value.trace()
    assert len(tr) == 1 and tr[0].iter == 1
    assert abs(tr[0].objective - z["gn_objective"][0]) <= 1e-6 * abs(z["gn_objective"][0])
