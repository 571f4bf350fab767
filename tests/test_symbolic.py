"""Host symbolic analysis through the C-ABI (CPU): bit-exact against the
reference's symbolic_analyze (core/cholesky.hpp:68-88) given the same ordering,
and structural invariants of the supernodal partition."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2503_08343_b200 as g
from conftest import golden_mat, load_golden


def _grid(gx, gy, radius=1):
    a = sp.diags([1.0] * (2 * radius + 1), list(range(-radius, radius + 1)), (gx, gx))
    b = sp.diags([1.0] * (2 * radius + 1), list(range(-radius, radius + 1)), (gy, gy))
    m = sp.kron(b, a).tocsc()
    m.sort_indices()
    return g.SparseMatrixCSC.from_scipy(m)


@pytest.mark.parametrize("fixture", ["corpus_acceptance.npz", "corpus_variance.npz"])
def test_symbolic_matches_reference_given_same_perm(lib_built, fixture):
    z = load_golden(fixture)
    for i in range(int(z["count"])):
        q = golden_mat(z, f"Q{i}")
        s = g.symbolic_analyze(q, z[f"perm{i}"])
        np.testing.assert_array_equal(s.parent, z[f"parent{i}"])
        np.testing.assert_array_equal(s.col_ptr, z[f"cpl{i}"])
        assert s.nnz_L == z[f"cpl{i}"][-1]
        np.testing.assert_array_equal(s.perm, z[f"perm{i}"])


def test_symbolic_matches_port_on_random_orders(lib_built, port):
    rng = np.random.default_rng(3)
    for q in [_grid(13, 11), _grid(20, 7, 2), _grid(30, 1)]:
        n = q.nrows
        for perm in [np.arange(n), rng.permutation(n), g.nd_order(q)]:
            s = g.symbolic_analyze(q, perm)
            parent, cpl = port.symbolic(n, q.col_ptr, q.row_idx, perm)
            np.testing.assert_array_equal(s.parent, parent)
            np.testing.assert_array_equal(s.col_ptr, cpl)


def test_nd_ordering_is_a_permutation_and_reduces_fill(lib_built, port):
    q = _grid(40, 40)
    n = q.nrows
    s = g.symbolic_analyze(q)  # ND, postordered
    assert sorted(s.perm.tolist()) == list(range(n))
    # the reported symbolic matches the port on the same (ND) permutation
    parent, cpl = port.symbolic(n, q.col_ptr, q.row_idx, s.perm)
    np.testing.assert_array_equal(s.parent, parent)
    np.testing.assert_array_equal(s.col_ptr, cpl)
    _, cpl_nat = port.symbolic(n, q.col_ptr, q.row_idx, np.arange(n))
    assert s.nnz_L < cpl_nat[-1]
    # postordered: every parent index exceeds its child
    assert np.all((s.parent == -1) | (s.parent > np.arange(n)))
    info = s.info
    assert info.n_supernodes <= n and info.nnz_l_padded >= info.nnz_l
    assert info.flops_sn >= info.flops_ref


def test_symbolic_rejects_bad_input(lib_built):
    q = _grid(4, 4)
    with pytest.raises(g.DimensionError):
        g.symbolic_analyze(q, np.zeros(16, np.int32))  # not a permutation
    bad = g.SparseMatrixCSC.from_arrays(3, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(g.DimensionError):
        g.symbolic_analyze(bad)


def test_symbolic_c1_matches_reference(lib_built):
    z = load_golden("c1_matern1d.npz")
    q = golden_mat(z, "Q_post")
    s = g.symbolic_analyze(q, z["perm_amd"])
    np.testing.assert_array_equal(s.col_ptr, z["L_cp"])


def test_symbolic_c2_matches_live_reference(lib_built, ref):
    b = ref.build("matern2d", [255, 10, 2, 1, 2000, 1002, 400, 0.05, 0, 2002, 0])
    qm = b.mat("Q_post")
    q = g.SparseMatrixCSC.from_arrays(qm.nrows, qm.ncols, qm.col_ptr, qm.row_idx, qm.values)
    perm = b.vec("perm_amd").astype(np.int32)
    parent, cpl = ref.symbolic(q.nrows, qm.col_ptr, qm.row_idx, perm)
    s = g.symbolic_analyze(q, perm)
    np.testing.assert_array_equal(s.parent, parent)
    np.testing.assert_array_equal(s.col_ptr, cpl)
    assert s.nnz_L == 8120088  # SURVEY §6 table, C2 under AMD
