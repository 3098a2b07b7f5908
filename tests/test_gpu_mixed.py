"""Acoustic-gravity block operator on B200 vs the reference (golden vectors of
feklab.operator.BlockOperator) and the oracle restatement (oracle/mixed.py).
Parity bar: max|y - y_ref| <= 1e-12 max|y_ref| per output block (normwise,
SURVEY.md §0.4); restriction maps bit-exact."""

import os

import numpy as np
import pytest

from oracle.mixed import MixedProblem

pytestmark = pytest.mark.gpu
TOL = 1e-12
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_mixed.npz")
CASES = ["m111", "m222", "m322_p2u1", "m232_p3u2", "m333_p6u5", "m443"]


def normwise(a, b):
    s = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (s if s > 0 else 1.0))


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLD)


def make(golden, name, **kw):
    from paper_2603_09038_b200 import MixedOperator, build_mesh

    m = golden[f"{name}_meta"]
    n = tuple(int(v) for v in m[:3])
    mesh = build_mesh(*n, extents=tuple(float(v) for v in m[3:6]))
    return MixedOperator(mesh, int(m[6]), int(m[7]), int(m[8]), rho=float(m[9]),
                         bulk_modulus=float(m[10]), coupling_scale=float(m[11]), **kw)


@pytest.mark.parametrize("strategy", ["FusedPA", "PA", "FusedMF", "MF"])
@pytest.mark.parametrize("name", CASES)
def test_apply_matches_reference(golden, name, strategy):
    from paper_2603_09038_b200 import MixedState

    op = make(golden, name, strategy=strategy)
    r = op.apply(MixedState(golden[f"{name}_u"], golden[f"{name}_p"]))
    assert normwise(r.u, golden[f"{name}_FusedPA_out_u"]) <= TOL
    assert normwise(r.p, golden[f"{name}_FusedPA_out_p"]) <= TOL
    assert op.counters.operator_applies == 1


@pytest.mark.parametrize("name", CASES)
def test_setup_data_matches_reference(golden, name):
    op = make(golden, name)
    assert np.array_equal(op.restriction_ids(), golden[f"{name}_gather"])
    lu, lp = op.lumped()
    assert normwise(lu, golden[f"{name}_lump_u"]) <= 1e-14
    assert normwise(lp, golden[f"{name}_lump_p"]) <= 1e-14


@pytest.mark.parametrize("name", CASES)
def test_fused_normal_mass_inverse_rk4(golden, name):
    from paper_2603_09038_b200 import MixedState

    op = make(golden, name)
    u, p = golden[f"{name}_u"], golden[f"{name}_p"]
    assert normwise(op.apply_fused_normal(u), golden[f"{name}_fused_normal"]) <= TOL
    mi = op.apply_mass_inverse(MixedState(u, p))
    assert normwise(mi.u, golden[f"{name}_minv_u"]) <= 1e-14
    assert normwise(mi.p, golden[f"{name}_minv_p"]) <= 1e-14
    st = op.rk4(MixedState(u, p), 1e-3, steps=2)
    assert normwise(st.u, golden[f"{name}_rk4_u"]) <= TOL
    assert normwise(st.p, golden[f"{name}_rk4_p"]) <= TOL
    assert op.counters.operator_applies == 8


@pytest.mark.parametrize("order_p", range(2, 9))
def test_every_order_vs_oracle(order_p):
    """Every compiled (order_p, order_p-1, order_p+1) on a ragged mesh with
    several batches per CTA, anisotropic extents, per-element coefficients."""
    from paper_2603_09038_b200 import MixedOperator, MixedState, build_mesh

    n = (7, 5, 6) if order_p <= 4 else (4, 3, 5)
    ext = (2.0, 1.0, 0.5)
    nel = n[0] * n[1] * n[2]
    rho = 1.0 + np.arange(nel) % 3
    P = MixedProblem(*n, order_p, order_p - 1, order_p + 1, extents=ext, rho=rho, bulk=2.0,
                     coupling_scale=0.75)
    op = MixedOperator(build_mesh(*n, extents=ext), order_p, order_p - 1, order_p + 1, rho=rho,
                       bulk_modulus=2.0, coupling_scale=0.75)
    rng = np.random.default_rng(order_p)
    u = rng.standard_normal(op.u_shape)
    p = rng.standard_normal(op.num_p)
    r = op.apply(MixedState(u, p))
    ru, rp = P.apply(u, p)
    assert normwise(r.u, ru) <= TOL
    assert normwise(r.p, rp) <= TOL
    assert normwise(op.apply_fused_normal(u), P.fused_normal(u)) <= TOL
    mf = MixedOperator(build_mesh(*n, extents=ext), order_p, order_p - 1, order_p + 1, rho=rho,
                       bulk_modulus=2.0, coupling_scale=0.75, strategy="FusedMF")
    r = mf.apply(MixedState(u, p))
    assert normwise(r.u, ru) <= TOL and normwise(r.p, rp) <= TOL
    lu, lp = op.lumped()
    assert normwise(lu, P.lump_u) <= 1e-14 and normwise(lp, P.lump_p) <= 1e-14


def test_large_mesh_many_batches():
    from paper_2603_09038_b200 import MixedOperator, MixedState, build_mesh

    n = (24, 20, 18)
    P = MixedProblem(*n)
    op = MixedOperator(build_mesh(*n))
    assert op.num_elements > 8 * op.launch[0] * op.launch[2] // 8
    rng = np.random.default_rng(5)
    u = rng.standard_normal(op.u_shape)
    p = rng.standard_normal(op.num_p)
    r = op.apply(MixedState(u, p))
    ru, rp = P.apply(u, p)
    assert normwise(r.u, ru) <= TOL and normwise(r.p, rp) <= TOL


def test_device_state_and_errors():
    import torch

    from paper_2603_09038_b200 import MixedOperator, MixedState, build_mesh

    op = MixedOperator(build_mesh(2, 2, 2))
    s = op.zero_state(device=True)
    s.p += 3.0
    r = op.apply(s)
    assert isinstance(r.u, torch.Tensor) and r.u.is_cuda
    # constant pressure: zero residual (test_operator.py:156-161)
    assert float(r.u.abs().max()) < 1e-13 and float(r.p.abs().max()) == 0.0
    bad = MixedState(np.zeros((3, 8, 27)), np.zeros(op.num_p))
    with pytest.raises(ValueError, match="do not match"):
        op.apply(bad)
    with pytest.raises(ValueError):
        MixedOperator(build_mesh(2, 2, 2), strategy="scalar")
    with pytest.raises(NotImplementedError):
        MixedOperator(build_mesh(2, 2, 2), order_u=2)
    assert MixedOperator(build_mesh(2, 2, 2), absorbing=True).absorbing  # now on the device path


def test_linear_pressure_gives_mass_weighted_unit_field():
    """test_operator.py:164-172 on the device operator."""
    from paper_2603_09038_b200 import MixedOperator, MixedState, build_mesh, h1_node_coords

    mesh = build_mesh(2, 3, 2)
    op = MixedOperator(mesh)
    coords = h1_node_coords(mesh, op.basis_p.nodes)
    r = op.apply(MixedState(np.zeros(op.u_shape), coords[:, 0].copy()))
    lu, _ = op.lumped()
    assert np.max(np.abs(r.u[0] - lu)) < 1e-13
    assert np.max(np.abs(r.u[1])) < 1e-13 and np.max(np.abs(r.u[2])) < 1e-13


@pytest.mark.parametrize("cfg", range(16))
@pytest.mark.parametrize("strategy", ["FusedPA", "FusedMF"])
@pytest.mark.parametrize("name", CASES)
def test_every_mixed_launch_config(golden, name, strategy, cfg, monkeypatch):
    """Every compiled geometry (FK_MIX_CFG, read at create): cfgs 0-3, their
    staged-output twins 4-7 (mix_pipe.cuh YS), single-X twins 8-11 (SX) and
    both 12-15 — both blocks, the composed normal operator (VB then TAU
    launches) and the matrix-free kernel."""
    from paper_2603_09038_b200 import MixedState

    monkeypatch.setenv("FK_MIX_CFG", str(cfg))
    op = make(golden, name, strategy=strategy)
    u, p = golden[f"{name}_u"], golden[f"{name}_p"]
    r = op.apply(MixedState(u, p))
    assert normwise(r.u, golden[f"{name}_FusedPA_out_u"]) <= TOL
    assert normwise(r.p, golden[f"{name}_FusedPA_out_p"]) <= TOL
    if strategy == "FusedPA":
        assert normwise(op.apply_fused_normal(u), golden[f"{name}_fused_normal"]) <= TOL


@pytest.mark.parametrize("cfg", range(16))
@pytest.mark.parametrize("name", ["m333_p6u5", "m443"])
def test_every_mixed_launch_config_multi_batch(golden, name, cfg, monkeypatch):
    """Persistent grid capped at 2 CTAs (FK_MAX_BLOCKS test hook): every CTA
    walks several batches, so the cross-batch prefetches (gid slots, the
    double or single X buffer, D after stage C) run, with a ragged last batch."""
    from paper_2603_09038_b200 import MixedState

    monkeypatch.setenv("FK_MIX_CFG", str(cfg))
    monkeypatch.setenv("FK_MAX_BLOCKS", "2")
    for strategy in ("FusedPA", "FusedMF"):
        op = make(golden, name, strategy=strategy)
        r = op.apply(MixedState(golden[f"{name}_u"], golden[f"{name}_p"]))
        assert normwise(r.u, golden[f"{name}_FusedPA_out_u"]) <= TOL
        assert normwise(r.p, golden[f"{name}_FusedPA_out_p"]) <= TOL
