"""P1 element assembly, lumping and Dirichlet folding
against the reference's own matrices (tests/golden/fem_p1.npz from
make_golden_fem.py: quadrature assembly of fem/assembly.hpp).

CPU: the host closed forms (gmrf_fem_assemble_host) reproduce the reference's
patterns exactly and its values to a few ulps. GPU: the device kernels
(gmrf_fem_assemble, csrc/fem_device.cu) equal the host closed forms bit for bit
and therefore sit at the same distance from the reference.
"""
import numpy as np
import pytest

from conftest import load_golden
from paper_2503_08343_b200.fem import assemble_p1
from paper_2503_08343_b200.regression import Mesh

ULPS = 8 * np.finfo(float).eps  # relative to the largest entry of the matrix


def _mesh(p):
    return Mesh.interval(int(p[1]), p[2], p[3]) if int(p[0]) == 1 else Mesh.unit_square(int(p[1]))


def _matrices(name, device):
    z = load_golden("fem_p1.npz")
    p = z[name + "_params"]
    mesh = _mesh(p)
    got = {}
    got["M"], got["lumped"] = assemble_p1(mesh, "mass", lumped=True, device=device)
    got["K"] = assemble_p1(mesh, "stiffness", p[4], p[5], p[6], device=device)
    if p[7]:
        got["M_c"], got["lumped_c"] = assemble_p1(mesh, "mass", dirichlet=True,
                                                  constrained_diag=p[8], lumped=True, device=device)
        got["K_c"] = assemble_p1(mesh, "stiffness", p[4], p[5], p[6], dirichlet=True,
                                 constrained_diag=1.0, device=device)
    return z, got


def _check_against_reference(name, device):
    z, got = _matrices(name, device)
    for key, m in got.items():
        if key.startswith("lumped"):
            ref = z[f"{name}_{key}"]
            assert np.max(np.abs(m - ref)) <= ULPS * np.max(np.abs(ref))
            continue
        np.testing.assert_array_equal(m.col_ptr, z[f"{name}_{key}_cp"])
        np.testing.assert_array_equal(m.row_idx, z[f"{name}_{key}_ri"])
        ref = z[f"{name}_{key}_v"]
        assert np.max(np.abs(m.values - ref)) <= ULPS * np.max(np.abs(ref)), key


@pytest.mark.parametrize("name", ["c4", "c1", "sq"])
def test_host_closed_forms_match_reference(name):
    _check_against_reference(name, device=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c4", "c1", "sq"])
def test_device_assembly_matches_reference_and_host(name):
    _check_against_reference(name, device=True)
    _, dev = _matrices(name, True)
    _, host = _matrices(name, False)
    for key in dev:
        a, b = dev[key], host[key]
        if key.startswith("lumped"):
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_array_equal(a.row_idx, b.row_idx)
            np.testing.assert_array_equal(a.values, b.values)  # bit for bit


@pytest.mark.gpu
def test_device_assembly_edge_meshes():
    for mesh in (Mesh.interval(1), Mesh.interval(2, -3.0, 5.0), Mesh.unit_square(1), Mesh.unit_square(2)):
        for which in ("mass", "stiffness"):
            a = assemble_p1(mesh, which, 0.7, 0.3 if mesh.dim == 1 else 0.0, 0.2 if mesh.dim == 1 else 0.0)
            b = assemble_p1(mesh, which, 0.7, 0.3 if mesh.dim == 1 else 0.0,
                            0.2 if mesh.dim == 1 else 0.0, device=False)
            np.testing.assert_array_equal(a.col_ptr, b.col_ptr)
            np.testing.assert_array_equal(a.row_idx, b.row_idx)
            np.testing.assert_array_equal(a.values, b.values)
