"""Host-side setup (paper_2603_09038_b200.fem) against the reference's golden data."""

import numpy as np
import pytest

from oracle import bp
from paper_2603_09038_b200 import fem
from paper_2603_09038_b200.operator import bytes_per_apply, flops_per_element, setup_pa_data


@pytest.mark.parametrize("d", range(2, 10))
def test_basis_bitwise(golden, d):
    for q in (d + 1, d):
        b = fem.Basis1D.nodal(d, q)
        assert np.array_equal(b.values, golden[f"basis_d{d}_q{q}_B"])
        assert np.array_equal(b.gradients, golden[f"basis_d{d}_q{q}_G"])
        assert np.array_equal(b.quad_weights, golden[f"basis_d{d}_q{q}_w"])
        assert np.array_equal(b.nodes, golden[f"basis_d{d}_q{q}_nodes"])


@pytest.mark.parametrize("n,d", [((2, 3, 4), 3), ((3, 3, 3), 5), ((4, 2, 3), 2), ((2, 2, 2), 9)])
def test_restriction_bitwise(golden, n, d):
    key = f"restr_{n[0]}x{n[1]}x{n[2]}_d{d}"
    r = fem.h1_restriction(fem.build_mesh(*n), d)
    assert r.gather_ids.dtype == np.int64
    assert np.array_equal(r.gather_ids, golden[key])
    assert np.array_equal(r.multiplicity(), golden[key + "_mult"])


def test_slab_rows_of_restriction():
    # rows [z0*nx*ny, z1*nx*ny) of the full map
    full = fem.h1_gather_ids(3, 2, 5, 4)
    part = fem.h1_gather_ids(3, 2, 5, 4, ez_range=(2, 4))
    assert np.array_equal(part, full[2 * 6: 4 * 6])


def test_node_coords(golden):
    mesh = fem.build_mesh(2, 3, 2, (2.0, 1.0, 0.5))
    c = fem.h1_node_coords(mesh, fem.Basis1D.nodal(4, 5).nodes)
    assert np.array_equal(c, golden["coords_2x3x2_d4"])


def test_mesh_geometry_matches_reference_conventions():
    # test_mesh.py:36-41
    m = fem.build_mesh(2, 1, 1, extents=(2.0, 1.0, 1.0))
    assert m.jacobian_det == 0.125
    assert np.allclose(m.jacobian_diag, [0.5, 0.5, 0.5])
    assert m.num_elements == 2
    assert m.vertices.shape == (12, 3)
    with pytest.raises(fem.GeometryError):
        fem.build_mesh(0, 1, 1)
    with pytest.raises(fem.GeometryError):
        fem.build_mesh(1, 1, 1, extents=(0.0, 1.0, 1.0))


def test_boundary_dofs_match_oracle():
    P = bp.Problem("diffusion", 3, 2, 4, 3)
    assert np.array_equal(fem.boundary_dofs(3, 2, 4, 4), P.boundary())


@pytest.mark.parametrize("p", range(1, 9))
def test_pa_data_matches_oracle_arithmetic(p):
    mesh = fem.build_mesh(3, 2, 2, (1.0, 2.0, 0.5))
    b = fem.Basis1D.nodal(p + 1, p + 2)
    P = bp.Problem("diffusion", 3, 2, 2, p, extents=(1.0, 2.0, 0.5))
    d = setup_pa_data(mesh, b, "diffusion").d
    assert np.array_equal(d[0], P.wdet * P.jinv[0] ** 2)
    assert np.array_equal(d[3], P.wdet * P.jinv[1] ** 2)
    assert np.array_equal(d[5], P.wdet * P.jinv[2] ** 2)
    assert not d[[1, 2, 4]].any()
    assert np.array_equal(setup_pa_data(mesh, b, "mass").d[0], P.wdet)


def test_roofline_accounting():
    # BP3 p=4 185.8 B/dof at 54^3, F/dof 516 (asymptotically)
    n, p = 54, 4
    d, q = p + 1, p + 2
    ndof, nel = (n * p + 1) ** 3, n ** 3
    assert abs(bytes_per_apply("diffusion", ndof, nel, d, q) / ndof - 185.8) < 3.0  # survey uses nel/ndof = 1/p^3
    assert flops_per_element("diffusion", d, q) == 2 * (4 * q * d ** 3 + 6 * q * q * d * d + 6 * q ** 3 * d) + 15 * q ** 3
    assert flops_per_element("mass", 3, 4) == 4 * (4 * 27 + 16 * 9 + 64 * 3) + 64
