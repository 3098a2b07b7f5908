"""The CPU oracle against the reference's golden vectors and known answers.

Pins oracle/ (the parity checker) before anything is compared with it:
golden vectors were produced by the real reference (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from oracle import bp
from _util import normwise

BP_CASES = (
    [("mass", (8, 8, 8), 2, None, (1.0, 1.0, 1.0), "bp1_8x8x8_p2")]
    + [("diffusion", (3, 3, 3), p, None, (1.0, 1.0, 1.0), f"bp3_3x3x3_p{p}") for p in range(1, 9)]
    + [("mass", (2, 2, 2), p, None, (1.0, 1.0, 1.0), f"bp1_2x2x2_p{p}") for p in range(1, 9)]
    + [("diffusion", (2, 3, 2), 3, None, (2.0, 1.0, 0.5), "bp3_2x3x2_p3_aniso"),
       ("diffusion", (3, 2, 4), 4, 5, (1.0, 1.0, 1.0), "bp3_3x2x4_p4_q5"),
       ("mass", (3, 2, 4), 4, 5, (1.0, 1.5, 1.0), "bp1_3x2x4_p4_q5")]
)


@pytest.mark.parametrize("d", range(2, 10))
def test_basis_tables_bitwise(golden, d):
    for q in (d + 1, d):
        B, G, w = bp.basis_tables(d, q)
        assert np.array_equal(B, golden[f"basis_d{d}_q{q}_B"])
        assert np.array_equal(G, golden[f"basis_d{d}_q{q}_G"])
        assert np.array_equal(w, golden[f"basis_d{d}_q{q}_w"])
        assert np.array_equal(bp.gll_points(d), golden[f"basis_d{d}_q{q}_nodes"])


@pytest.mark.parametrize("n,d", [((2, 3, 4), 3), ((3, 3, 3), 5), ((4, 2, 3), 2), ((2, 2, 2), 9)])
def test_gather_ids_bitwise(golden, n, d):
    key = f"restr_{n[0]}x{n[1]}x{n[2]}_d{d}"
    ids = bp.gather_ids(*n, d)
    assert ids.dtype == np.int64
    assert np.array_equal(ids, golden[key])
    mult = bp.scatter_add(ids, np.ones(ids.shape), bp.num_dofs(*n, d))
    assert np.array_equal(mult, golden[key + "_mult"])


@pytest.mark.parametrize("kind,n,p,q,ext,key", BP_CASES)
def test_batched_oracle_bitwise(golden, kind, n, p, q, ext, key):
    P = bp.Problem(kind, *n, p, q, ext)
    y = P.apply(golden[key + "_x"])
    assert np.array_equal(y, golden[key + "_y"])
    assert np.array_equal(P.diagonal(), golden[key + "_diag"])


@pytest.mark.parametrize("kind,n,p,q,ext,key", [c for c in BP_CASES if c[2] in (1, 2, 4)])
def test_per_element_oracle_bitwise(golden, kind, n, p, q, ext, key):
    P = bp.Problem(kind, *n, p, q, ext)
    assert np.array_equal(P.apply(golden[key + "_x"], batched=False), golden[key + "_y"])


@pytest.mark.parametrize("key,n,p", [("cg_3x3x3_p3", (3, 3, 3), 3), ("cg_2x2x3_p5", (2, 2, 3), 5)])
def test_pcg_history_bitwise(golden, key, n, p):
    P = bp.Problem("diffusion", *n, p)
    hist_ref = golden[key + "_hist"]
    x, hist = P.pcg(golden[key + "_b"], iters=len(hist_ref) - 1)
    assert np.array_equal(hist, hist_ref)
    assert np.array_equal(x, golden[key + "_x"])


# -- reference known answers (feklab tests) restated on the oracle -------------


def test_contract_identity_rotates_indices():
    # test_tensor.py:108-117 — identity contraction only rotates the indices
    x = np.random.default_rng(0).standard_normal(4 * 3 * 2)
    out, ext = bp.contract_cyclic(np.eye(4), x, (4, 3, 2))
    assert ext == (3, 2, 4)
    assert np.array_equal(out.reshape(ext, order="F"),
                          x.reshape((4, 3, 2), order="F").transpose(1, 2, 0))


def test_partition_of_unity_and_constant_gradient():
    # test_tensor.py:166-169, :255-259
    for d in range(2, 10):
        B, G, _ = bp.basis_tables(d, d + 1)
        ones = np.ones(d ** 3)
        assert np.max(np.abs(bp.chain((B, B, B), ones, (d, d, d)) - 1.0)) < 1e-12
        for r in range(3):
            g = bp.chain([G if s == r else B for s in range(3)], ones, (d, d, d))
            assert np.max(np.abs(g)) < 1e-11


def test_kronecker_oracle():
    # test_tensor.py:172-179 (Kronecker matrices on F-order vectors)
    rng = np.random.default_rng(4)
    d, q = 4, 5
    B = rng.standard_normal((q, d))
    x = rng.standard_normal(d ** 3)
    y = bp.chain((B, B, B), x, (d, d, d))
    K = np.kron(B, np.kron(B, B))
    assert normwise(y, K @ x) <= 1e-12


def test_transpose_is_adjoint():
    # test_tensor.py:190-201, :213-226
    rng = np.random.default_rng(8)
    for _ in range(50):
        d, q = 4, 5
        B = rng.standard_normal((q, d))
        x, yv = rng.standard_normal(d ** 3), rng.standard_normal(q ** 3)
        lhs = bp.chain((B, B, B), x, (d, d, d)) @ yv
        rhs = x @ bp.chain((B.T, B.T, B.T), yv, (q, q, q))
        assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


def _interp_x(p, nx, extent):
    h = extent / nx
    xs = np.empty(nx * p + 1)
    for e in range(nx):
        xs[e * p: e * p + p + 1] = e * h + (bp.gll_points(p + 1) + 1.0) * 0.5 * h
    return xs


def test_physics_identities():
    # 1'M1 = volume; f'Af = volume for f = interpolant of x
    for p in (2, 4, 6):
        for ext in ((1.0, 1.0, 1.0), (2.0, 1.0, 0.5)):
            vol = ext[0] * ext[1] * ext[2]
            M = bp.Problem("mass", 2, 3, 2, p, extents=ext)
            one = np.ones(M.ndof)
            assert abs(one @ M.apply(one) - vol) < 1e-13
            A = bp.Problem("diffusion", 2, 3, 2, p, extents=ext)
            f = np.tile(_interp_x(p, 2, ext[0]), (3 * p + 1) * (2 * p + 1))
            assert abs(f @ A.apply(f) - vol) < 1e-12
            assert np.max(np.abs(A.apply(one))) < 1e-12
