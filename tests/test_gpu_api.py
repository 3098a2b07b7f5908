"""Boundary behaviour of the Python operator API (advisor findings, round 1)."""

import numpy as np
import pytest

from oracle import bp
from paper_2603_09038_b200 import Counters, MixedOperator, MixedState, PAOperator, cg_solve, fem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_host_buffers_are_validated():
    op = PAOperator(fem.build_mesh(2, 2, 2), 3)
    n = op.num_dofs
    x = np.random.default_rng(0).standard_normal(n)
    for bad in (np.empty(n, np.float32), np.empty(n - 1), np.empty(2 * n)[::2]):
        with pytest.raises(ValueError):
            op.apply(x, out=bad)
        with pytest.raises((ValueError, TypeError)):
            op.apply_host(x, bad)
    with pytest.raises(ValueError):
        op.apply_host(x[:-1], np.empty(n))
    with pytest.raises(ValueError):
        op.apply_host(torch.zeros(n, dtype=torch.float64, device="cuda"), np.empty(n))
    out = np.empty(n)
    assert op.apply(x, out=out) is out
    assert np.allclose(out, bp.Problem("diffusion", 2, 2, 2, 3).apply(x), rtol=0, atol=1e-12 * np.abs(out).max())


def test_set_config_failure_keeps_kernel():
    op = PAOperator(fem.build_mesh(3, 3, 3), 4)
    before = (op.variant, op.info.cfg, op.launch)
    with pytest.raises(NotImplementedError):
        op.set_config("eo", 999)
    assert (op.variant, op.info.cfg, op.launch) == before


def test_cg_zero_rhs_and_all_essential_mesh_do_not_nan():
    op = PAOperator(fem.build_mesh(3, 3, 3), 3, dirichlet=True)
    x, h = cg_solve(op, np.zeros(op.num_dofs), iters=10)
    assert len(h) == 1 and h[0] == 0.0 and np.all(x == 0.0)
    op1 = PAOperator(fem.build_mesh(1, 1, 1), 1, dirichlet=True)  # every dof essential
    b = np.random.default_rng(0).standard_normal(op1.num_dofs)
    x1, h1 = cg_solve(op1, b * 0.0, iters=5)
    assert np.all(np.isfinite(x1)) and np.all(np.isfinite(h1))


def test_counter_semantics_match_reference():
    """feklab counts d_reads only for the PA strategies (operator.py:280-286;
    tests/test_operator.py:271-289: MF reads no D) and one apply per call;
    cg_solve counts the applies actually run."""
    mesh = fem.build_mesh(2, 2, 2)
    c_pa, c_mf = Counters(), Counters()
    pa = PAOperator(mesh, 3, strategy="PA", counters=c_pa)
    mf = PAOperator(mesh, 3, strategy="MF", counters=c_mf)
    x = torch.randn(pa.num_dofs, dtype=torch.float64, device="cuda")
    pa.apply(x)
    mf.apply(x)
    assert c_mf.d_reads == 0 and c_pa.d_reads > 0
    assert c_pa.operator_applies == c_mf.operator_applies == 1 and c_pa.flops == c_mf.flops
    c = Counters()
    op = PAOperator(fem.build_mesh(3, 3, 3), 3, dirichlet=True, counters=c)
    b = np.random.default_rng(0).standard_normal(op.num_dofs)
    b[bp.Problem("diffusion", 3, 3, 3, 3).boundary()] = 0
    _, h = cg_solve(op, b, iters=500, rtol=1e-3)
    assert c.operator_applies == len(h) - 1 < 500


def test_mixed_rejects_unsymmetric_tables(monkeypatch):
    """The block operator's kernel folds the 1D tables even-odd; tables that
    are not mirror-symmetric (to the 128-ulp rounding of Basis1D.nodal) are
    refused instead of silently symmetrised."""
    from paper_2603_09038_b200 import mixed
    from paper_2603_09038_b200.fem import Basis1D

    real = Basis1D.nodal

    def skewed(d, q, *a, **k):
        b = real(d, q, *a, **k)
        v = np.array(b.values)
        v[0, 0] += 1e-9
        return Basis1D(b.num_dofs_1d, b.num_quad_1d, v, np.array(b.gradients), b.nodes,
                       b.quad_points, b.quad_weights)

    monkeypatch.setattr(mixed.Basis1D, "nodal", staticmethod(skewed))
    with pytest.raises(NotImplementedError, match="symmetric"):
        MixedOperator(fem.build_mesh(2, 2, 2), 4, 3, 5)


@pytest.mark.parametrize("kind,p", [("diffusion", 3), ("diffusion", 6), ("mass", 4)])
def test_diagonal_closed_form_and_general_kernel_agree(kind, p):
    """The box diagonal is one separable closed-form pass (fk_setup.cuh
    diag_box_kernel); a caller-supplied gather map takes the general
    element-wise kernel.  Both match the oracle's assembled diagonal."""
    n = (4, 3, 5)
    mesh = fem.build_mesh(*n, extents=(2.0, 1.0, 0.5))
    P = bp.Problem(kind, *n, p, extents=(2.0, 1.0, 0.5))
    ref = P.diagonal()
    box = PAOperator(mesh, p, kind=kind).diagonal().cpu().numpy()
    gen = PAOperator(mesh, p, kind=kind, restriction=fem.h1_restriction(mesh, p + 1)).diagonal().cpu().numpy()
    scale = np.abs(ref).max()
    assert np.abs(box - ref).max() <= 1e-13 * scale
    assert np.abs(gen - ref).max() <= 1e-13 * scale


def test_mixed_apply_fills_host_out_in_place():
    op = MixedOperator(fem.build_mesh(2, 2, 2))
    rng = np.random.default_rng(0)
    s = MixedState(rng.standard_normal(op.u_shape), rng.standard_normal(op.num_p))
    ref = op.apply(s)
    out = MixedState(np.empty(op.u_shape), np.empty(op.num_p))
    assert op.apply(s, out=out) is out
    # u is stored directly (bitwise); p is scattered with atomics (order varies)
    assert np.array_equal(out.u, ref.u)
    assert np.max(np.abs(out.p - ref.p)) <= 1e-14 * np.max(np.abs(ref.p))
    with pytest.raises(ValueError):
        op.apply(s, out=MixedState(np.empty(op.u_shape, np.float32), np.empty(op.num_p)))
    with pytest.raises(ValueError, match="do not match"):
        op.apply(s, out=MixedState(np.empty((3, 1, 1)), np.empty(op.num_p)))
    dev = MixedState(torch.empty(op.u_shape, dtype=torch.float64, device="cuda"),
                     torch.empty(op.num_p, dtype=torch.float64, device="cuda"))
    assert op.apply(s, out=dev) is dev
    assert np.array_equal(dev.u.cpu().numpy(), ref.u)
    assert np.max(np.abs(dev.p.cpu().numpy() - ref.p)) <= 1e-14 * np.max(np.abs(ref.p))
