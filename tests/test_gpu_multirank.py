"""The multi-rank library path (z-slabs) executed for real.

Groups of nranks = 2..4 rank PROCESSES (tests/_rankpool.py) share cuda:0,
each with its own CUDA context, exactly as one process per GPU on an 8-GPU
box: the peer-memory transport of fk_comm.cu with the mailboxes mapped
through CUDA IPC (bootstrap over gloo), the put / flag / add kernels, the
rank-ordered slot allreduce, apply_overlapped (nz_local >= 3), the owned-dof
dots, slab Dirichlet faces, the diagonal exchange and the CUDA-graph-captured
CG.  Results are compared with the single-process CPU oracle on the same
global mesh (normwise 1e-12; CG: identical iteration counts, histories within
1e-8 h_0, as tests/test_gpu_parity.py), and shared interface planes must be
bit-identical on both neighbours.
"""

import numpy as np
import pytest

from _util import PARITY_TOL, normwise
from oracle import bp
from paper_2603_09038_b200 import Comm, PAOperator, fem, parallel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


_POOLS = {}


@pytest.fixture(scope="module")
def pools():
    from _rankpool import RankPool

    def get(world):
        if world not in _POOLS:
            _POOLS[world] = RankPool(world)
        return _POOLS[world]

    yield get
    for p in _POOLS.values():
        p.close()
    _POOLS.clear()


def assemble(parts, ndof, plane, key):
    y = np.zeros(ndof)
    for r, part in enumerate(parts):
        if r > 0:
            assert np.array_equal(parts[r - 1][key][-plane:], part[key][:plane]), \
                f"shared plane of ranks {r - 1}/{r} differs"
        y[part["lo"]:part["hi"]] = part[key]
    return y


CASES = [
    # kind, mesh, p, world  (nz_local = 1, 2, 3 and ragged slabs)
    ("diffusion", (3, 2, 4), 3, 4),     # nz_local 1: plain exchange
    ("diffusion", (3, 3, 4), 4, 2),     # nz_local 2
    ("diffusion", (2, 3, 9), 3, 3),     # nz_local 3: overlapped apply
    ("diffusion", (2, 2, 7), 6, 2),     # ragged 4/3, p=6 (configs[4] order)
    ("mass", (3, 2, 6), 5, 3),
    ("diffusion", (4, 3, 10), 4, 4),    # ragged 3/3/2/2
]


@pytest.mark.parametrize("kind,n,p,world", CASES)
@pytest.mark.parametrize("dirichlet", [False, True])
def test_multirank_apply_matches_oracle(pools, kind, n, p, world, dirichlet):
    res = pools(world).run("apply", kind=kind, n=n, p=p, dirichlet=dirichlet)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(7).standard_normal(P.ndof)
    ref = P.constrained_apply(x, P.boundary()) if dirichlet else P.apply(x)
    y = assemble(res, P.ndof, parallel.plane_size(n[0], n[1], p), "y")
    assert normwise(y, ref) <= PARITY_TOL
    for r in res:  # the three repeated applies agree to rounding
        assert normwise(r["all"][0], r["y"]) <= 1e-15


@pytest.mark.parametrize("world", [2, 3, 4])
def test_multirank_dot_owned_dofs(pools, world):
    vals = pools(world).run("dot", n=(3, 2, 8), p=3)
    P = bp.Problem("diffusion", 3, 2, 8, 3)
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(P.ndof), rng.standard_normal(P.ndof)
    ref = float(a @ b)
    for v in vals:
        assert v == vals[0]  # every rank holds the same bits (slot sums in rank order)
        assert abs(v[0] - ref) <= 1e-13 * np.sqrt(float(a @ a) * float(b @ b))


@pytest.mark.parametrize("kind,n,p,world", [("diffusion", (3, 2, 6), 4, 3), ("mass", (2, 3, 4), 3, 2)])
def test_multirank_diagonal(pools, kind, n, p, world):
    res = pools(world).run("diagonal", kind=kind, n=n, p=p)
    P = bp.Problem(kind, *n, p)
    ref = P.diagonal()
    ref[P.boundary()] = 1.0
    assert normwise(assemble(res, P.ndof, parallel.plane_size(n[0], n[1], p), "d"), ref) <= PARITY_TOL


CG_CASES = [
    ("diffusion", (3, 3, 6), 3, 2, "auto", 60),
    ("diffusion", (3, 3, 6), 3, 3, "auto", 60),
    ("diffusion", (2, 3, 8), 4, 4, "auto", 50),
    ("diffusion", (3, 2, 9), 4, 3, "auto", 50),     # nz_local 3: overlapped apply inside the graph
    ("diffusion", (2, 2, 6), 6, 2, "auto", 40),     # p=6
    ("diffusion", (3, 2, 6), 4, 2, "mf", 50),       # matrix-free operator
    ("mass", (3, 3, 4), 2, 2, "auto", 30),
]


@pytest.mark.parametrize("kind,n,p,world,variant,iters", CG_CASES)
def test_multirank_cg_matches_oracle(pools, kind, n, p, world, variant, iters):
    res = pools(world).run("cg", kind=kind, n=n, p=p, iters=iters, variant=variant)
    P = bp.Problem(kind, *n, p)
    b = np.random.default_rng(0).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    xr, hr = P.pcg(b, iters=iters)
    for r in res:
        assert len(r["h"]) == len(hr)
        assert np.array_equal(r["h"], res[0]["h"])  # identical scalars on every rank
        assert np.max(np.abs(r["h"] - hr)) <= 1e-8 * hr[0]
        assert r["applies"] == iters
    x = assemble(res, P.ndof, parallel.plane_size(n[0], n[1], p), "x")
    assert normwise(x, xr) <= 1e-8


def test_multirank_cg_rtol_stops_every_rank_together(pools):
    res = pools(3).run("cg", kind="diffusion", n=(3, 3, 6), p=3, iters=200, rtol=1e-6, seed=1)
    P = bp.Problem("diffusion", 3, 3, 6, 3)
    b = np.random.default_rng(1).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    _, hr = P.pcg(b, iters=200, rtol=1e-6)
    assert all(len(r["h"]) == len(hr) for r in res) and len(hr) < 201
    assert all(r["applies"] == len(hr) - 1 for r in res)


def test_multirank_matches_single_gpu(pools):
    """Interior dofs of a slab see the same element contributions as the
    single-GPU apply; only shared planes add two partial sums in another order."""
    n, p = (3, 3, 8), 4
    res = pools(2).run("apply", kind="diffusion", n=n, p=p)
    single = PAOperator(fem.build_mesh(*n), p)
    x = np.random.default_rng(7).standard_normal(single.num_dofs)
    ref = single.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    y = assemble(res, single.num_dofs, parallel.plane_size(n[0], n[1], p), "y")
    assert normwise(y, ref) <= 1e-15
    single.close()


def test_deterministic_multirank_cg_bitwise(pools):
    """Verification mode across ranks: colour-ordered slabs, rank-ordered
    reductions — two solves are bit-identical (history and solution)."""
    kw = dict(kind="diffusion", n=(3, 3, 8), p=4, iters=40, seed=5, deterministic=True)
    a = pools(3).run("cg", **kw)
    b = pools(3).run("cg", **kw)
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["h"], rb["h"]) and np.array_equal(ra["x"], rb["x"])
    P = bp.Problem("diffusion", 3, 3, 8, 4)
    bb = np.random.default_rng(5).standard_normal(P.ndof)
    bb[P.boundary()] = 0.0
    _, hr = P.pcg(bb, iters=40)
    assert np.max(np.abs(a[0]["h"] - hr)) <= 1e-8 * hr[0]


def test_deterministic_multirank_apply_bitwise(pools):
    res = pools(2).run("apply", kind="diffusion", n=(4, 3, 6), p=3, deterministic=True, reps=4)
    for r in res:
        for y in r["all"]:
            assert np.array_equal(y, r["all"][0])


def test_plane_capacity_is_checked():
    comm = Comm(0, 1, 0, transport="p2p", plane_cap=10)
    with pytest.raises(ValueError, match="does not match"):
        PAOperator(fem.build_mesh(3, 3, 4), 3, comm=comm)
    comm.close()


def test_multirank_long_cg_protocol_stress(pools):
    """300 graph-replayed iterations on 3 ranks: ~900 exchanges and slot
    reductions (double-buffered by parity) without a host in the loop; the
    history still tracks the oracle and every rank agrees bitwise."""
    iters = 300
    res = pools(3).run("cg", kind="diffusion", n=(2, 2, 6), p=3, iters=iters, seed=11)
    P = bp.Problem("diffusion", 2, 2, 6, 3)
    b = np.random.default_rng(11).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    _, hr = P.pcg(b, iters=iters)
    for r in res:
        assert np.array_equal(r["h"], res[0]["h"]) and len(r["h"]) == len(hr)
    # relative to the initial residual; late iterations sit at rounding level
    assert np.max(np.abs(res[0]["h"] - hr)) <= 1e-8 * hr[0]


@pytest.mark.parametrize("kind,n,p,q,ext,world,variant", [
    ("diffusion", (3, 2, 6), 3, 4, (2.0, 1.0, 0.5), 3, "auto"),   # q = p+1, anisotropic box
    ("diffusion", (2, 3, 6), 4, 6, (1.0, 3.0, 2.0), 2, "mf"),     # matrix-free, anisotropic
    ("mass", (3, 3, 6), 2, 3, (0.5, 1.0, 1.5), 3, "auto"),
    ("diffusion", (2, 2, 8), 5, 7, (1.0, 1.0, 4.0), 4, "dmma"),   # batched DMMA kernel across ranks
])
def test_multirank_apply_anisotropic_and_q(pools, kind, n, p, q, ext, world, variant):
    res = pools(world).run("apply", kind=kind, n=n, p=p, q=q, extents=ext, variant=variant,
                           dirichlet=True)
    P = bp.Problem(kind, *n, p, q, extents=ext)
    x = np.random.default_rng(7).standard_normal(P.ndof)
    ref = P.constrained_apply(x, P.boundary())
    y = assemble(res, P.ndof, parallel.plane_size(n[0], n[1], p), "y")
    assert normwise(y, ref) <= PARITY_TOL
