"""GPU: batched posterior sampling (sample_direct, gmrf.hpp:173/182) and the
Rao-Blackwellized Monte Carlo variance estimator (rbmc_variance, gmrf.hpp:
213-240) against the unmodified reference (oracle/_ref) on the same Q, mean,
permutation and seed. The z draws are identical (same Rng stream, core/rng.hpp);
the samples then differ only by the solves' rounding, so they agree to ~1e-13
relative. Acceptance criterion 10 (acceptance.cpp:612-666): RBMC with 2000
samples within 5% of the Takahashi variances."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2503_08343_b200 as g

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def grid(nx, ny, diag=4.2):
    t = sp.diags([-1.0, -1.0], [-1, 1], (nx, nx))
    k = sp.kron(sp.eye(ny), t) + sp.kron(sp.diags([-1.0, -1.0], [-1, 1], (ny, ny)), sp.eye(nx))
    q = (k + diag * sp.eye(nx * ny)).tocsc()
    q.sort_indices()
    return g.SparseMatrixCSC.from_scipy(q)


def tridiag(n):
    q = sp.diags([-1.0, 2.2, -1.0], [-1, 0, 1], (n, n)).tocsc()
    q.sort_indices()
    return g.SparseMatrixCSC.from_scipy(q)


@pytest.mark.parametrize("ns", [1, 16, 37])
def test_sample_direct_matches_reference(ref, ns):
    q = grid(40, 35)
    f = g.cholesky_factor(q)
    mu = np.random.default_rng(3).standard_normal(q.nrows)
    x = g.sample_direct(f, mu, ns, 2002)
    xr = ref.sample_direct(q.nrows, q.col_ptr, q.row_idx, q.values, f.perm, mu, ns, 2002)
    assert x.shape == (q.nrows, ns)
    assert rel(x, xr) <= 1e-12


def test_rbmc_matches_reference(ref):
    q = grid(30, 30, diag=4.05)
    f = g.cholesky_factor(q)
    mu = np.linspace(-1.0, 1.0, q.nrows)
    v = g.rbmc_variance(f, q, mu, 50, 12345)
    vr = ref.rbmc_variance(q.nrows, q.col_ptr, q.row_idx, q.values, f.perm, mu, 50, 12345)
    assert rel(v, vr) <= 1e-10


@pytest.mark.parametrize("q", [tridiag(400), grid(20, 20)], ids=["tridiag400", "grid20"])
def test_rbmc_vs_takahashi_acceptance(q):
    # acceptance.cpp:643-650: 2000 samples, seed 12345, zero mean, tol 5%
    f = g.cholesky_factor(q)
    exact = g.takahashi_diagonal(f)
    est = g.rbmc_variance(f, q, np.zeros(q.nrows), 2000, 12345)
    assert rel(est, exact) <= 0.05


def test_rbmc_errors():
    q = tridiag(50)
    f = g.cholesky_factor(q)
    with pytest.raises(g.ContractError):
        g.rbmc_variance(f, q, np.zeros(50), 1, 1)
    bad = g.SparseMatrixCSC(q.nrows, q.ncols, q.col_ptr, q.row_idx, q.values.copy())
    bad.values[q.col_ptr[7]:q.col_ptr[8]][q.row_idx[q.col_ptr[7]:q.col_ptr[8]] == 7] = -1.0
    with pytest.raises(g.NumericalError):
        g.rbmc_variance(f, bad, np.zeros(50), 4, 1)
