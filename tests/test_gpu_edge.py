"""Edge cases through the C-ABI (GPU): empty and 1×1 systems, decoupled
(diagonal / disconnected) patterns, many right-hand sides (> one 16-wide
pass), lower/upper modes against the C restatement, refactor with new values,
non-SPD inside a larger matrix, and wide supernodes (> several 64-chunks)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2503_08343_b200 as g

pytestmark = pytest.mark.gpu


def csc(m):
    m = sp.csc_matrix(m)
    m.sort_indices()
    return g.SparseMatrixCSC.from_scipy(m)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300)


def test_empty_and_one_by_one():
    q0 = g.SparseMatrixCSC.from_arrays(0, 0, [0], [], [])
    f0 = g.cholesky_factor(q0)
    assert g.solve(f0, np.zeros(0)).shape == (0,)
    assert g.takahashi_diagonal(f0).shape == (0,)
    q1 = g.SparseMatrixCSC.from_arrays(1, 1, [0, 1], [0], [9.0])
    f1 = g.cholesky_factor(q1)
    assert f1.L.values[0] == pytest.approx(3.0)
    assert g.solve(f1, [18.0])[0] == pytest.approx(2.0)
    assert g.takahashi_diagonal(f1)[0] == pytest.approx(1.0 / 9.0)


def test_decoupled_patterns():
    rng = np.random.default_rng(4)
    d = rng.uniform(1, 5, 500)
    f = g.cholesky_factor(csc(sp.diags(d)))
    np.testing.assert_allclose(g.takahashi_diagonal(f), 1.0 / d, rtol=1e-14)
    # two disconnected grid components plus isolated nodes
    a = sp.diags([-1.0, 4.0, -1.0], [-1, 0, 1], (40, 40))
    m = sp.block_diag([a, sp.eye(7) * 2.0, a * 2.0]).tocsc()
    q = csc(m)
    f = g.cholesky_factor(q)
    b = rng.standard_normal(m.shape[0])
    assert rel(g.solve(f, b), np.linalg.solve(m.toarray(), b)) <= 1e-13
    np.testing.assert_allclose(g.takahashi_diagonal(f), np.diag(np.linalg.inv(m.toarray())),
                               rtol=1e-12)


def test_many_rhs_and_modes_vs_port(port):
    gx = 70
    a = sp.diags([-1.0, 4.2, -1.0], [-1, 0, 1], (gx, gx))
    m = (sp.kron(sp.eye(gx), a) + sp.kron(sp.diags([-1.0, -1.0], [-1, 1], (gx, gx)), sp.eye(gx)))
    q = csc(m)
    n = q.nrows
    f = g.cholesky_factor(q)
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, f.perm)
    rng = np.random.default_rng(9)
    b = rng.standard_normal((n, 37))  # 16 + 16 + 5 right-hand sides
    for mode in (0, 1, 2):
        x = g.solve_triangular(f, b, mode)
        xo = port.solve(n, lcp, lri, lv, f.perm, mode, b)
        assert rel(x, xo) <= 1e-12, mode


def test_refactor_new_values_and_failure():
    gx = 30
    a = sp.diags([-1.0, 4.0, -1.0], [-1, 0, 1], (gx, gx))
    m = (sp.kron(sp.eye(gx), a) + sp.kron(sp.diags([-1.0, -1.0], [-1, 1], (gx, gx)), sp.eye(gx)))
    q = csc(m)
    sym = g.symbolic_analyze(q)
    f = g.CholeskyFactor(sym)
    rng = np.random.default_rng(2)
    for shift in (0.5, 3.0):
        v = q.values.copy()
        dmask = np.zeros_like(v, bool)
        for j in range(q.ncols):
            for p in range(q.col_ptr[j], q.col_ptr[j + 1]):
                dmask[p] = q.row_idx[p] == j
        v[dmask] += shift
        f.refactor(v)
        mm = sp.csc_matrix((v, q.row_idx, q.col_ptr), shape=m.shape)
        b = rng.standard_normal(q.nrows)
        assert rel(g.solve(f, b), np.linalg.solve(mm.toarray(), b)) <= 1e-12
    # make one diagonal entry strongly negative: reported in original numbering
    v = q.values.copy()
    k = 417
    p = q.col_ptr[k] + np.searchsorted(q.row_idx[q.col_ptr[k]:q.col_ptr[k + 1]], k)
    v[p] = -50.0
    with pytest.raises(g.NotPositiveDefiniteError) as e:
        f.refactor(v)
    assert 0 <= e.value.index() < q.nrows
    # the factor recovers on the next valid refactor
    f.refactor(q.values)
    b = np.ones(q.nrows)
    assert rel(g.solve(f, b), np.linalg.solve(m.toarray(), b)) <= 1e-12


def test_wide_supernodes_dense_block(port):
    # a dense 300x300 SPD block coupled to a chain: one supernode of ~5 chunks
    rng = np.random.default_rng(1)
    a = rng.standard_normal((300, 300))
    dense = a @ a.T + 300 * np.eye(300)
    chain = sp.diags([-1.0, 3.0, -1.0], [-1, 0, 1], (200, 200)).toarray()
    m = np.zeros((500, 500))
    m[:300, :300] = dense
    m[300:, 300:] = chain
    m[299, 300] = m[300, 299] = -0.5
    q = csc(m)
    f = g.cholesky_factor(q)
    info = f.sym.info
    assert info.max_front >= 300
    n = q.nrows
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, f.perm)
    assert rel(f.L.values, lv) <= 1e-12
    inv = np.linalg.inv(m)
    np.testing.assert_allclose(g.takahashi_diagonal(f), np.diag(inv), rtol=1e-10)
    s = g.takahashi_selected_inverse(f).to_scipy().tocoo()
    assert np.abs(s.data - inv[s.row, s.col]).max() <= 1e-12
    # triangle solves through the multi-CTA wide kernels (w > 256)
    b = rng.standard_normal((n, 21))
    for mode in (0, 1, 2):
        for k in (1, 4, 21):
            x = g.solve_triangular(f, b[:, :k], mode)
            xo = port.solve(n, lcp, lri, lv, f.perm, mode, b[:, :k])
            assert rel(x, xo) <= 1e-12, (mode, k)


def test_wide_supernodes_many_per_level(port):
    # 3-D 7-point grid: several wide separators on the same tree levels, plus a
    # dense 1100-wide block (18 row blocks in one cooperative launch)
    gx = 22
    a = sp.diags([-1.0, 6.3, -1.0], [-1, 0, 1], (gx, gx))
    off = sp.diags([-1.0, -1.0], [-1, 1], (gx, gx))
    i1 = sp.eye(gx)
    grid = (sp.kron(sp.kron(i1, i1), a) + sp.kron(sp.kron(i1, off), i1) +
            sp.kron(sp.kron(off, i1), i1))
    rng = np.random.default_rng(7)
    d = rng.standard_normal((1100, 1100)) / 40.0
    dense = d @ d.T + 2.0 * np.eye(1100)
    m = sp.block_diag([grid, sp.csc_matrix(dense)]).tolil()
    m[0, grid.shape[0]] = m[grid.shape[0], 0] = -0.25
    m = m.tocsc()
    q = csc(m)
    f = g.cholesky_factor(q)
    n = q.nrows
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, f.perm)
    assert bad < 0
    assert rel(f.L.values, lv) <= 1e-12
    b = rng.standard_normal((n, 19))
    for mode in (0, 1, 2):
        for k in (1, 3, 19):
            x = g.solve_triangular(f, b[:, :k], mode)
            xo = port.solve(n, lcp, lri, lv, f.perm, mode, b[:, :k])
            assert rel(x, xo) <= 1e-12, (mode, k)
    # repeated solves are bit-identical (fixed accumulation order)
    x1 = g.solve(f, b[:, 0])
    x2 = g.solve(f, b[:, 0])
    assert np.array_equal(x1, x2)
    xs = g.solve(f, b[:, 0])
    assert rel(m @ xs, b[:, 0]) <= 1e-10


def _supernodes(sym):
    import ctypes as C
    from paper_2503_08343_b200 import _capi
    ns = int(sym.info.n_supernodes)
    first = np.zeros(ns + 1, np.int32)
    rows = np.zeros(ns, np.int32)
    p32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    assert _capi.load().gmrf_symbolic_supernodes(sym._h, p32(first), p32(rows), None, None) == 0
    return np.diff(first), rows


@pytest.mark.parametrize("seed", [0, 1])
def test_small_front_buckets_and_warp_solves(port, seed):
    # dense leaf blocks of width w all coupled to one separator of size s: each
    # leaf is one front with rows = w + s. (w, s) picks every small-front kernel
    # (rows <= 32, <= 64, and 64 < rows <= 96 with w <= 16 / 32 / 64 / > 64) and
    # the warp-per-supernode solves (w <= 64, rows <= 128)
    rng = np.random.default_rng(seed)
    shapes = [(10, 12), (20, 30), (12, 70), (24, 60), (48, 40), (70, 20), (40, 80)]
    blocks, cols, n0 = [], [], 0
    sep = 90
    for w, s in shapes:
        blocks.append((n0, w, s))
        n0 += w
    n = n0 + sep
    m = np.zeros((n, n))
    for b0, w, s in blocks:
        a = rng.standard_normal((w, w))
        m[b0:b0 + w, b0:b0 + w] = a @ a.T + w * np.eye(w)
        c = rng.standard_normal((s, w)) * 0.1
        m[n0:n0 + s, b0:b0 + w] = c
        m[b0:b0 + w, n0:n0 + s] = c.T
    d = rng.standard_normal((sep, sep))
    m[n0:, n0:] += d @ d.T / sep + 40.0 * np.eye(sep)
    q = csc(m)
    f = g.cholesky_factor(q, np.arange(n))  # leaves first, separator last
    widths, rows = _supernodes(f.sym)
    got = {(int(w), int(r)) for w, r in zip(widths, rows)}
    for w, s in shapes:
        assert (w, w + s) in got, (w, s, sorted(got))
    lcp, lri, lv, bad = port.cholesky(n, q.col_ptr, q.row_idx, q.values, f.perm)
    assert bad < 0
    assert rel(f.L.values, lv) <= 1e-12
    b = rng.standard_normal((n, 6))
    for mode in (0, 1, 2):
        for k in (1, 4, 6):
            x = g.solve_triangular(f, b[:, :k], mode)
            xo = port.solve(n, lcp, lri, lv, f.perm, mode, b[:, :k])
            assert rel(x, xo) <= 1e-12, (mode, k)
    np.testing.assert_allclose(g.takahashi_diagonal(f), np.diag(np.linalg.inv(m)), rtol=1e-10)
    # a non-positive pivot inside a row-sweep small front reports its original index
    m2 = m.copy()
    b0, w, s = blocks[4]  # (48, 40): k_small_front_rows<64>
    m2[b0 + 30, b0 + 30] = -5.0
    with pytest.raises(g.NotPositiveDefiniteError) as e:
        g.cholesky_factor(csc(m2), np.arange(n))
    assert e.value.index() == b0 + 30
