"""Host (no GPU) parts of the Matérn regression pipeline against the
reference's own outputs on the seeded C1/C2 inputs (tests/golden/make_golden.py):
the point observation operator (eval_basis / locate, fem/space.hpp:67-109,
376-394) must be bit-identical — same element choice on ties, same shape
values."""
import numpy as np
import pytest

from conftest import golden_mat, load_golden
from paper_2503_08343_b200.regression import Mesh, point_observation_operator


@pytest.mark.parametrize("fixture,mesh", [("c1_matern1d.npz", Mesh.interval(999)),
                                          ("c2_matern2d.npz", Mesh.unit_square(255))])
def test_point_operator_bit_exact(lib_built, fixture, mesh):
    z = load_golden(fixture)
    a_ref = golden_mat(z, "A")
    a = point_observation_operator(mesh, z["points"])
    assert (a.nrows, a.ncols) == (a_ref.nrows, a_ref.ncols)
    np.testing.assert_array_equal(a.col_ptr, a_ref.col_ptr)
    np.testing.assert_array_equal(a.row_idx, a_ref.row_idx)
    np.testing.assert_array_equal(a.values, a_ref.values)


def test_point_operator_rejects_outside_points(lib_built):
    from paper_2503_08343_b200 import ContractError
    with pytest.raises(ContractError):
        point_observation_operator(Mesh.interval(10), [0.5, 1.5])
    with pytest.raises(ContractError):
        point_observation_operator(Mesh.unit_square(4), [0.5, 0.5, -0.1, 0.2])


def test_point_operator_edges_and_nodes(lib_built):
    # points on nodes / cell edges / the diagonal: every row sums to 1
    pts = np.array([0.0, 0.0, 1.0, 1.0, 0.25, 0.25, 0.5, 0.125, 0.75, 1.0])
    a = point_observation_operator(Mesh.unit_square(4), pts).to_scipy()
    np.testing.assert_allclose(np.asarray(a.sum(axis=1)).ravel(), 1.0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("config,fixture", [(1, "c1_matern1d.npz"), (2, "c2_matern2d.npz")])
def test_seeded_inputs_match_reference_draws(lib_built, config, fixture):
    """The product regenerates the reference's seeded C1/C2 inputs (Rng stream,
    SURVEY §8(d) draw order): points bit-exact, data within an ulp (libm sin/cos)."""
    from paper_2503_08343_b200.regression import seeded_inputs
    z = load_golden(fixture)
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(config)
    np.testing.assert_array_equal(pts, z["points"])
    np.testing.assert_allclose(y, z["y"], rtol=0, atol=4e-16)
    assert np.all(z["noise"] == lam)
