"""Pins the C restatement (oracle/gmrf_oracle.c) to the reference.

CPU-only. The restatement must reproduce the reference bit for bit on the
reference's own seeded corpora (tests/oracles.hpp spd_corpus, fixtures made by
tests/golden/make_golden.py from the unmodified reference), and satisfy the
reference's known-answer tests (test_factorization.cpp, test_takahashi_cg.cpp).
"""
import numpy as np
import pytest

from conftest import golden_mat, load_golden


def _dense(m):
    d = np.zeros((m.nrows, m.ncols))
    for j in range(m.ncols):
        for p in range(m.col_ptr[j], m.col_ptr[j + 1]):
            d[m.row_idx[p], j] = m.values[p]
    return d


@pytest.mark.parametrize("fixture", ["corpus_acceptance.npz", "corpus_variance.npz"])
def test_port_bit_exact_on_reference_corpus(port, fixture):
    z = load_golden(fixture)
    for i in range(int(z["count"])):
        q = golden_mat(z, f"Q{i}")
        n = q.nrows
        perm = z[f"perm{i}"]
        parent, cpl = port.symbolic(n, q.col_ptr, q.row_idx, perm)
        np.testing.assert_array_equal(parent, z[f"parent{i}"])
        np.testing.assert_array_equal(cpl, z[f"cpl{i}"])
        lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, perm)
        assert bad == -1
        np.testing.assert_array_equal(lcp, z[f"L{i}_cp"])
        np.testing.assert_array_equal(lri, z[f"L{i}_ri"])
        np.testing.assert_array_equal(lv, z[f"L{i}_v"])  # bit-exact
        b = z[f"b{i}"]
        np.testing.assert_array_equal(port.solve(n, lcp, lri, lv, perm, 2, b)[:, 0], z[f"x{i}"])
        np.testing.assert_array_equal(port.solve(n, lcp, lri, lv, perm, 0, b)[:, 0], z[f"xl{i}"])
        np.testing.assert_array_equal(port.solve(n, lcp, lri, lv, perm, 1, b)[:, 0], z[f"xu{i}"])
        np.testing.assert_array_equal(port.takahashi_diag(n, lcp, lri, lv, perm), z[f"var{i}"])


def test_port_selected_inverse_matches_reference_pattern(port):
    z = load_golden("corpus_acceptance.npz")
    for i in range(0, 50, 7):
        q = golden_mat(z, f"Q{i}")
        n = q.nrows
        perm = z[f"perm{i}"]
        lcp, lri, lv, _ = port.cholesky(n, q.col_ptr, q.row_idx, q.values, perm)
        sv = port.takahashi(n, lcp, lri, lv)
        s = golden_mat(z, f"S{i}")
        for j in range(n):
            for p in range(lcp[j], lcp[j + 1]):
                assert s.coeff(perm[lri[p]], perm[j]) == sv[p]


def test_port_known_answers(port):
    # cholesky of 4I is 2I (test_factorization.cpp:102-108)
    cp = np.arange(4, dtype=np.int64)
    ri = np.arange(3, dtype=np.int32)
    lcp, lri, lv, bad = port.cholesky(3, cp, ri, np.full(3, 4.0), np.arange(3))
    assert bad == -1 and np.all(lv == 2.0)
    # 2x2 closed form (test_factorization.cpp:110-116)
    cp = np.array([0, 2, 4], np.int64)
    ri = np.array([0, 1, 0, 1], np.int32)
    v = np.array([4.0, 2.0, 2.0, 3.0])
    lcp, lri, lv, bad = port.cholesky(2, cp, ri, v, np.arange(2))
    np.testing.assert_allclose(lv, [2.0, 1.0, np.sqrt(2.0)])
    x = port.solve(2, lcp, lri, lv, np.arange(2), 2, np.array([1.0, 0.0]))[:, 0]
    np.testing.assert_allclose(x, [0.375, -0.25], rtol=1e-12)
    # indefinite input reports original index 1 (test_factorization.cpp:145-154)
    cp = np.arange(4, dtype=np.int64)
    _, _, _, bad = port.cholesky(3, cp, ri[:3], np.array([2.0, -1.0, 3.0]), np.arange(3))
    assert bad == 1
    # takahashi of (4I)^-1 is 0.25 (test_takahashi_cg.cpp:27-31)
    cp = np.arange(6, dtype=np.int64)
    lcp, lri, lv, _ = port.cholesky(5, cp, np.arange(5, dtype=np.int32), np.full(5, 4.0),
                                    np.arange(5))
    np.testing.assert_allclose(port.takahashi_diag(5, lcp, lri, lv, np.arange(5)), 0.25)


def test_port_tridiagonal_takahashi_vs_dense(port):
    # test_takahashi_cg.cpp:33-39: tridiagonal(6, 2, -1), ≤1e-12 vs the dense inverse
    n = 6
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(2.0)
        if i + 1 < n:
            rows += [i, i + 1]; cols += [i + 1, i]; vals += [-1.0, -1.0]
    import scipy.sparse as sp
    m = sp.csc_matrix((vals, (rows, cols)), shape=(n, n))
    m.sort_indices()
    perm = np.arange(n)[::-1].copy()
    lcp, lri, lv, _ = port.cholesky(n, m.indptr, m.indices, m.data, perm)
    d = port.takahashi_diag(n, lcp, lri, lv, perm)
    np.testing.assert_allclose(d, np.diag(np.linalg.inv(m.toarray())), atol=1e-12)


def test_port_c2_mean_and_samples_match_reference(port):
    """C2 posterior (2D Matérn, n = 65,536): from the reference's Q_post bits and
    AMD permutation the port reproduces the reference's mean and its first two
    samples (z from the Rng mirror, core/rng.hpp). The variances (≈70 s of
    single-core Takahashi) are checked on the GPU against the same fixture."""
    import paper_2503_08343_b200 as g
    z = load_golden("c2_matern2d.npz")
    q = golden_mat(z, "Q_post")
    n = q.nrows
    perm = z["perm_amd"]
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, perm)
    assert bad == -1
    rhs = golden_mat(z, "A").to_scipy().T @ (z["noise"] * z["y"])
    mean = port.solve(n, lcp, lri, lv, perm, 2, rhs)[:, 0]
    assert np.linalg.norm(mean - z["mean_post"]) <= 1e-13 * np.linalg.norm(z["mean_post"])
    zz = g.Rng(2002).normal_vector(2 * n).reshape(2, n)
    ss = z["samples"].reshape(2, n)
    for k in range(2):
        w = port.solve(n, lcp, lri, lv, perm, 1, zz[k])[:, 0]
        x = np.empty(n)
        x[perm] = w
        np.testing.assert_allclose(x + z["mean_post"], ss[k], rtol=0, atol=1e-13)


def test_port_c1_pipeline_matches_reference(port):
    """C1 posterior: the port reproduces the reference's mean,
    Takahashi variances and sample draws from the reference's Q_post bits."""
    z = load_golden("c1_matern1d.npz")
    q = golden_mat(z, "Q_post")
    a = golden_mat(z, "A")
    n = q.nrows
    perm = z["perm_amd"]
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, perm)
    assert bad == -1
    np.testing.assert_array_equal(lv, z["L_v"])
    rhs = a.to_scipy().T @ (z["noise"] * z["y"])
    # gmrf.hpp:157-162 (prior mean 0, b = 0): the reference forms rhs with
    # matvec_transpose; summation order can differ by an ulp.
    mean = port.solve(n, lcp, lri, lv, perm, 2, rhs)[:, 0]
    np.testing.assert_allclose(mean, z["mean_post"], rtol=1e-13, atol=1e-13)
    np.testing.assert_array_equal(port.takahashi_diag(n, lcp, lri, lv, perm), z["var_post"])
    zz = z["z"].reshape(8, n)
    ss = z["samples"].reshape(8, n)
    for k in range(8):
        w = port.solve(n, lcp, lri, lv, perm, 1, zz[k])[:, 0]
        x = np.empty(n)
        x[perm] = w
        np.testing.assert_allclose(x + z["mean_post"], ss[k], rtol=0, atol=1e-14)


def test_port_against_live_reference(port, ref):
    """Fresh inputs (not in the fixtures): 2D grid + random SPD, natural/AMD/reverse orders."""
    rng = np.random.default_rng(7)
    import scipy.sparse as sp
    g = 9
    lap = sp.kron(sp.eye(g), sp.diags([-1, 4.1, -1], [-1, 0, 1], (g, g))) + \
        sp.kron(sp.diags([-1, -1], [-1, 1], (g, g)), sp.eye(g))
    a = sp.random(40, 40, 0.1, random_state=3)
    for m in [lap.tocsc(), (a.T @ a + 20 * sp.eye(40)).tocsc()]:
        m.sort_indices()
        n = m.shape[0]
        for perm in [np.arange(n), ref.amd_order(n, m.indptr, m.indices), rng.permutation(n)]:
            f = ref.factor(n, m.indptr, m.indices, m.data, perm)
            rcp, rri, rv, _ = f.L()
            lcp, lri, lv, _ = port.cholesky(n, m.indptr, m.indices, m.data, perm)
            np.testing.assert_array_equal(lv, rv)
            np.testing.assert_array_equal(port.takahashi_diag(n, lcp, lri, lv, perm),
                                          f.takahashi_diag())


def test_allen_cahn_restatement_pins():
    """The C5 residual is absent from the reference; its CPU
    restatement must pass the reference's finite-difference Jacobian check
    pattern (acceptance.cpp:503-608, tolerance 1e-5) and drive the reference
    gauss_newton to convergence on the fixture."""
    z = load_golden("c5_allen_cahn_8x8x16.npz")
    assert z["fd_rel_err"][0] <= 1e-5
    assert len(z["gn_objective"]) >= 2 and z["gn_objective"][-1] < z["gn_objective"][0]
    assert np.all(z["var_post"] > 0)
