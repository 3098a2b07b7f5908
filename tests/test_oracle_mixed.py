"""Oracle for the acoustic-gravity block operator pinned to the reference's
own outputs (tests/golden/golden_mixed.npz, made by make_golden_mixed.py
from feklab.operator.BlockOperator / rk4_step)."""

import os

import numpy as np
import pytest

from oracle.mixed import MixedProblem

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_mixed.npz")
CASES = ["m111", "m222", "m322_p2u1", "m232_p3u2", "m333_p6u5", "m443"]


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLD)


def problem(golden, name):
    m = golden[f"{name}_meta"]
    n = tuple(int(v) for v in m[:3])
    return MixedProblem(*n, order_p=int(m[6]), order_u=int(m[7]), q=int(m[8]),
                        extents=tuple(m[3:6]), rho=m[9], bulk=m[10], coupling_scale=m[11])


@pytest.mark.parametrize("name", CASES)
def test_apply_bitexact(golden, name):
    P = problem(golden, name)
    u, p = golden[f"{name}_u"], golden[f"{name}_p"]
    ou, op = P.apply(u, p)
    for strat in ("PA", "FusedPA"):
        assert np.array_equal(ou, golden[f"{name}_{strat}_out_u"]), strat
        assert np.array_equal(op, golden[f"{name}_{strat}_out_p"]), strat


@pytest.mark.parametrize("name", CASES)
def test_restriction_and_lumped_mass(golden, name):
    P = problem(golden, name)
    assert np.array_equal(P.ids, golden[f"{name}_gather"])
    assert np.array_equal(P.lump_u, golden[f"{name}_lump_u"])
    assert np.array_equal(P.lump_p, golden[f"{name}_lump_p"])
    mu, mp = P.mass_inverse(golden[f"{name}_u"], golden[f"{name}_p"])
    assert np.array_equal(mu, golden[f"{name}_minv_u"])
    assert np.array_equal(mp, golden[f"{name}_minv_p"])


@pytest.mark.parametrize("name", CASES)
def test_fused_normal_and_rk4(golden, name):
    P = problem(golden, name)
    u, p = golden[f"{name}_u"], golden[f"{name}_p"]
    assert np.array_equal(P.fused_normal(u), golden[f"{name}_fused_normal"])
    for _ in range(2):
        u, p = P.rk4_step(u, p, 1e-3)
    assert np.array_equal(u, golden[f"{name}_rk4_u"])
    assert np.array_equal(p, golden[f"{name}_rk4_p"])


def test_velocity_block_is_negative_transpose():
    """operator.py tests :184-190: A_pu = -A_up^T (probed on a 1-element mesh)."""
    P = MixedProblem(1, 1, 1, 2, 1, 3)
    nu = 3 * P.du ** 3
    A = np.zeros((nu + P.ndof_p, nu + P.ndof_p))
    for j in range(A.shape[1]):
        v = np.zeros(A.shape[1])
        v[j] = 1.0
        ou, op = P.apply(v[:nu].reshape(3, 1, -1), v[nu:])
        A[:, j] = np.concatenate([ou.ravel(), op])
    assert np.max(np.abs(A[nu:, :nu] + A[:nu, nu:].T)) <= 1e-13 * np.max(np.abs(A))
