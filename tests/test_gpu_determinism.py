"""Verification mode (fk_op_desc.deterministic) and the
reference's determinism contract.

The reference scatters with sequential np.add.at (mesh.py:133-137) and pins
bitwise determinism of its operators (tests/test_tensor.py:320-326); the
default B200 apply scatters with FP64 atomics, whose order varies run to
run.  With deterministic=True the elements run in 8-colour order (one launch
per colour, no two elements of a colour share a node), so every dof sums its
contributions in colour order: y, the Jacobi diagonal and whole CG solves
must be bit-identical across runs — single rank and multi-rank — and still
match the oracle.
"""

import numpy as np
import pytest

from _util import PARITY_TOL, normwise
from oracle import bp
from paper_2603_09038_b200 import PAOperator, cg_solve, fem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


CASES = [("diffusion", (5, 4, 3), 4), ("diffusion", (7, 6, 5), 3), ("mass", (6, 5, 4), 2),
         ("diffusion", (3, 3, 3), 8), ("diffusion", (1, 1, 1), 2), ("mass", (9, 2, 3), 6),
         ("diffusion", (2, 5, 7), 5), ("diffusion", (4, 4, 4), 1)]


@pytest.mark.parametrize("kind,n,p", CASES)
@pytest.mark.parametrize("variant", ["auto", "mf", "dfma"])
def test_deterministic_apply_parity_and_bitwise_repeat(kind, n, p, variant):
    op = PAOperator(fem.build_mesh(*n), p, kind=kind, deterministic=True, variant=variant)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(1).standard_normal(P.ndof)
    xd = dev(x)
    ys = [op.apply(xd).cpu().numpy() for _ in range(5)]
    assert normwise(ys[0], P.apply(x)) <= PARITY_TOL
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])
    # restriction hook still reports the reference's element order
    assert np.array_equal(op.restriction_ids(), bp.gather_ids(*n, p + 1))


def test_deterministic_large_mesh_bitwise_across_runs():
    """Many CTAs and batches (contended dofs in the default mode): 54x40x30 p=4."""
    n, p = (54, 40, 30), 4
    op = PAOperator(fem.build_mesh(*n), p, deterministic=True)
    x = torch.randn(op.num_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    y0 = op.apply(x)
    for _ in range(4):
        assert torch.equal(op.apply(x), y0)
    ref = PAOperator(fem.build_mesh(*n), p)
    assert normwise(y0.cpu().numpy(), ref.apply(x).cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("p", [3, 4, 6])
def test_deterministic_diagonal_and_cg_bitwise(p):
    n = (4, 3, 5)
    op = PAOperator(fem.build_mesh(*n), p, dirichlet=True, deterministic=True)
    P = bp.Problem("diffusion", *n, p)
    d0 = op.diagonal().cpu().numpy()
    ref = P.diagonal()
    ref[P.boundary()] = 1.0
    assert normwise(d0, ref) <= PARITY_TOL
    assert np.array_equal(op.diagonal().cpu().numpy(), d0)
    b = np.random.default_rng(0).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    runs = [cg_solve(op, b, iters=60) for _ in range(3)]
    _, hr = P.pcg(b, iters=60)
    for x, h in runs:
        assert np.array_equal(h, runs[0][1]) and np.array_equal(x, runs[0][0])
    assert np.max(np.abs(runs[0][1] - hr)) <= 1e-8 * hr[0]


def test_deterministic_rejects_user_map_and_closed_form_cfg():
    mesh = fem.build_mesh(3, 3, 3)
    with pytest.raises(NotImplementedError, match="deterministic"):
        PAOperator(mesh, 3, deterministic=True, restriction=fem.h1_restriction(mesh, 4))
    op = PAOperator(mesh, 4, deterministic=True)
    before = (op.variant, op.info.cfg)
    with pytest.raises(NotImplementedError, match="closed-form"):
        op.set_config("eo", 35)
    assert (op.variant, op.info.cfg) == before  # failed selection leaves the kernel in place
