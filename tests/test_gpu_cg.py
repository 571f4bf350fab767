"""GPU: conjugate gradients (cg_solve, core/cg.hpp:39-105) and CG posterior
sampling (sample_cg, gmrf.hpp:188-202) against the unmodified reference and
the factorization: acceptance criterion 1's CG part (acceptance.cpp:92-105:
Jacobi CG at rtol 1e-10 within 1e-6 of the Cholesky solution on
spd_corpus(50, 20240817)), iteration counts vs the reference, the reference's
sample_cg unit cases (test_gmrf.cpp:242-289) and error behaviour."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2503_08343_b200 as g
from conftest import golden_mat, load_golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def test_cg_corpus_vs_cholesky_and_reference(ref):
    z = load_golden("corpus_acceptance.npz")
    rng = np.random.default_rng(5)
    worst, iters_gap = 0.0, 0
    for i in range(int(z["count"])):
        q = golden_mat(z, f"Q{i}")
        n = q.nrows
        b = rng.standard_normal(n)
        direct = g.solve(g.cholesky_factor(q), b)
        cfg = g.CGConfig(rtol=1e-10, max_iter=100 * n, preconditioner=g.Preconditioner.kJacobi)
        r = g.cg_solve(q, b, None, cfg)
        assert r.converged
        worst = max(worst, rel(r.x, direct))
        xr, it_r, res_r, conv_r = ref.cg_solve(n, q.col_ptr, q.row_idx, q.values, b, 1e-10, 0.0,
                                               100 * n, True)
        assert conv_r
        assert rel(r.x, xr) <= 1e-8
        iters_gap = max(iters_gap, abs(r.iterations - it_r))
    assert worst <= 1e-6
    # same recurrence and stopping rule: the iteration counts agree (reductions
    # are summed in a different order, which may move a borderline stop by one)
    assert iters_gap <= 1


def test_cg_unpreconditioned_and_warm_start(ref):
    n = 300
    q = g.SparseMatrixCSC.from_scipy(sp.diags([-1.0, 2.3, -1.0], [-1, 0, 1], (n, n)).tocsc())
    b = np.sin(np.arange(n))
    r = g.cg_solve(q, b, None, g.CGConfig(rtol=1e-12))
    xr, it_r, _, _ = ref.cg_solve(n, q.col_ptr, q.row_idx, q.values, b, 1e-12)
    assert r.converged and abs(r.iterations - it_r) <= 1 and rel(r.x, xr) <= 1e-10
    r2 = g.cg_solve(q, b, r.x, g.CGConfig(rtol=1e-12))  # already converged: 0 iterations
    assert r2.converged and r2.iterations == 0
    r3 = g.cg_solve(q, b, None, g.CGConfig(rtol=1e-14, max_iter=3))
    assert not r3.converged and r3.iterations == 3


def test_cg_errors():
    q = g.SparseMatrixCSC.from_scipy(sp.diags([1.0, -1.0, 1.0]).tocsc())
    with pytest.raises(g.NumericalError):  # non-positive curvature (cg.hpp:74-76)
        g.cg_solve(q, np.array([0.0, 1.0, 0.0]))
    with pytest.raises(g.ContractError):
        g.cg_solve(q, np.ones(3), None, g.CGConfig(rtol=0.0))
    with pytest.raises(g.DimensionError):
        g.cg_solve(q, np.ones(4))


def test_sample_cg_reference_cases():
    # test_gmrf.cpp:242-253: identity Q and S
    n = 5
    mu = np.arange(n) * 0.5 - 1.0
    eye = g.SparseMatrixCSC.from_scipy(sp.eye(n).tocsc())
    np.testing.assert_allclose(g.sample_cg(eye, eye, mu, np.zeros(n)), mu)
    zz = np.array([0.3, -1.2, 2.0, 0.1, -0.7])
    np.testing.assert_allclose(g.sample_cg(eye, eye, np.zeros(n), zz), zz, rtol=1e-9)
    # general: mean + Q⁻¹ S z against the factorization
    m = 80
    qs = sp.diags([-0.8, 2.0, -0.8], [-1, 0, 1], (m, m)).tocsc()
    s_sqrt = sp.csc_matrix(np.linalg.cholesky(qs.toarray()))
    q = g.SparseMatrixCSC.from_scipy(qs)
    s = g.SparseMatrixCSC.from_scipy(s_sqrt)
    z = np.random.default_rng(2).standard_normal(m)
    u = g.sample_cg(q, s, np.ones(m), z, g.CGConfig(rtol=1e-12))
    np.testing.assert_allclose(u - 1.0, g.solve(g.cholesky_factor(q), s_sqrt @ z), rtol=1e-9,
                               atol=1e-10)
    with pytest.raises(g.DimensionError):
        g.sample_cg(q, s, np.ones(m), np.zeros(m + 1))
    with pytest.raises(g.NumericalError):  # CG did not reach tolerance
        g.sample_cg(q, s, np.ones(m), z, g.CGConfig(rtol=1e-14, max_iter=2))
