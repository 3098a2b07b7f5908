"""Parity of the CUDA path (through the C-ABI) with the CPU oracle / reference.

Bars:
* integer restriction maps: bit-exact;
* PA data: bit-exact (same arithmetic as setup_pa_data / the reference);
* operator apply: max|y - y_ref| <= 1e-12 * max|y_ref|  (PARITY_TOL);
* CG: identical iteration counts, |h_k - h_ref,k| <= 1e-8 * h_0.
"""

import numpy as np
import pytest

from _util import PARITY_TOL, normwise
from oracle import bp
from paper_2603_09038_b200 import PAOperator, cg_solve, fem, setup_pa_data

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


def make(kind, n, p, q=None, ext=(1.0, 1.0, 1.0), **kw):
    mesh = fem.build_mesh(*n, extents=ext)
    return PAOperator(mesh, p, q, kind=kind, **kw)


def dev(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")


VARIANTS = ["dfma", "dmma", "eo", "mf"]

GOLDEN_CASES = (
    [("mass", (8, 8, 8), 2, None, (1.0, 1.0, 1.0), "bp1_8x8x8_p2")]
    + [("diffusion", (3, 3, 3), p, None, (1.0, 1.0, 1.0), f"bp3_3x3x3_p{p}") for p in range(1, 9)]
    + [("mass", (2, 2, 2), p, None, (1.0, 1.0, 1.0), f"bp1_2x2x2_p{p}") for p in range(1, 9)]
    + [("diffusion", (2, 3, 2), 3, None, (2.0, 1.0, 0.5), "bp3_2x3x2_p3_aniso"),
       ("diffusion", (3, 2, 4), 4, 5, (1.0, 1.0, 1.0), "bp3_3x2x4_p4_q5"),
       ("mass", (3, 2, 4), 4, 5, (1.0, 1.5, 1.0), "bp1_3x2x4_p4_q5")]
)


def _variant_ok(op, variant):
    try:
        op.set_variant(variant)
        return True
    except NotImplementedError:
        return False


# -- integer maps and setup ----------------------------------------------------


@pytest.mark.parametrize("n,d", [((2, 3, 4), 3), ((3, 3, 3), 5), ((4, 2, 3), 2), ((2, 2, 2), 9)])
def test_restriction_bit_exact(golden, n, d):
    op = make("diffusion", n, d - 1)
    ids = op.restriction_ids()
    assert ids.dtype == np.int64
    assert np.array_equal(ids, golden[f"restr_{n[0]}x{n[1]}x{n[2]}_d{d}"])


def test_restriction_bit_exact_large():
    # BP3 p=4 config mesh (54^3): device closed form vs host closed form
    op = make("diffusion", (54, 54, 54), 4)
    assert np.array_equal(op.restriction_ids(), fem.h1_gather_ids(54, 54, 54, 5))


def test_restriction_from_reference_map(golden):
    # an explicit gather map (Restriction object) instead of the closed form
    ids = golden["restr_3x3x3_d5"]
    op = make("diffusion", (3, 3, 3), 4, restriction=fem.Restriction(int(ids.max()) + 1, ids))
    assert np.array_equal(op.restriction_ids(), ids)


@pytest.mark.parametrize("kind", ["mass", "diffusion"])
@pytest.mark.parametrize("p", [1, 4, 8])
def test_pa_data_bit_exact(kind, p):
    mesh = fem.build_mesh(3, 2, 2, extents=(1.0, 2.0, 0.5))
    op = PAOperator(mesh, p, kind=kind)
    ref = setup_pa_data(mesh, op.basis, kind).d
    got = op.pa_data()
    assert got.shape == (12, ref.shape[0], (p + 2) ** 3)
    assert np.array_equal(got, np.broadcast_to(ref, got.shape))


# -- operator apply --------------------------------------------------------------


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("kind,n,p,q,ext,key", GOLDEN_CASES)
def test_apply_matches_reference_golden(golden, variant, kind, n, p, q, ext, key):
    op = make(kind, n, p, q, ext)
    if not _variant_ok(op, variant):
        pytest.skip(f"{variant} not compiled for p={p} q={q}")
    y = op.apply(dev(golden[key + "_x"])).cpu().numpy()
    assert normwise(y, golden[key + "_y"]) <= PARITY_TOL


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("kind", ["mass", "diffusion"])
@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("qoff", [1, 2])
def test_apply_matches_oracle_all_orders(variant, kind, p, qoff):
    n = (3, 2, 4) if p <= 4 else (2, 2, 3)
    op = make(kind, n, p, p + qoff, (1.0, 0.7, 1.3))
    if not _variant_ok(op, variant):
        pytest.skip(f"{variant} not compiled for p={p} q={p + qoff}")
    P = bp.Problem(kind, *n, p, p + qoff, (1.0, 0.7, 1.3))
    x = np.random.default_rng(p).standard_normal(P.ndof)
    y = op.apply(dev(x)).cpu().numpy()
    assert normwise(y, P.apply(x)) <= PARITY_TOL


LAUNCH_CONFIGS = ([("dfma", c) for c in range(7)] + [("dmma", c) for c in range(15)]
                  + [("eo", c) for c in range(62)] + [("mf", c) for c in range(11)])


@pytest.mark.parametrize("variant,cfg", LAUNCH_CONFIGS)
@pytest.mark.parametrize("kind", ["mass", "diffusion"])
@pytest.mark.parametrize("p", range(1, 9))
def test_every_launch_config(variant, cfg, kind, p):
    """Every compiled (variant, E, T) geometry, incl. the Dirichlet-bit path and
    meshes whose element count does not fill the last batch."""
    n = (5, 3, 3) if p <= 4 else (3, 2, 3)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(p).standard_normal(P.ndof)
    for dirichlet in (False, True):
        op = make(kind, n, p, dirichlet=dirichlet)
        try:
            op.set_config(variant, cfg)
        except NotImplementedError as ex:  # geometry exceeds 227 KB smem at this order
            pytest.skip(str(ex))
        y = op.apply(dev(x)).cpu().numpy()
        ref = P.constrained_apply(x, P.boundary()) if dirichlet else P.apply(x)
        assert normwise(y, ref) <= PARITY_TOL, (op.launch, dirichlet)


@pytest.mark.parametrize("variant,cfg", LAUNCH_CONFIGS)
@pytest.mark.parametrize("kind", ["mass", "diffusion"])
@pytest.mark.parametrize("p", range(1, 9))
def test_every_launch_config_multi_batch(variant, cfg, kind, p, monkeypatch):
    """Persistent grid capped at 3 CTAs (FK_MAX_BLOCKS test hook): every CTA
    walks several batches, so the cross-batch prefetches (x gather one batch
    ahead, gather-id slots two ahead, PA data to smem / L2 / registers) and the
    ping-pong buffers are exercised, with a ragged last batch."""
    monkeypatch.setenv("FK_MAX_BLOCKS", "3")
    n = (5, 4, 3) if p <= 4 else (3, 3, 3)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(p + 7).standard_normal(P.ndof)
    for dirichlet in (False, True):
        op = make(kind, n, p, dirichlet=dirichlet)
        try:
            op.set_config(variant, cfg)
        except NotImplementedError as ex:
            pytest.skip(str(ex))
        if (variant, cfg) != ("dfma", 5):  # dfma5: one batch per CTA, no persistent grid
            assert op.launch[2] <= 3
        y = op.apply(dev(x)).cpu().numpy()
        ref = P.constrained_apply(x, P.boundary()) if dirichlet else P.apply(x)
        assert normwise(y, ref) <= PARITY_TOL, (op.launch, dirichlet)


@pytest.mark.parametrize("n", [(1, 1, 1), (3, 1, 2), (1, 5, 1), (7, 3, 5)])
@pytest.mark.parametrize("p", [1, 4, 7])
def test_ragged_meshes(n, p):
    # element counts that do not fill the last CTA batch
    for kind in ("mass", "diffusion"):
        op = make(kind, n, p)
        P = bp.Problem(kind, *n, p)
        x = np.random.default_rng(1).standard_normal(P.ndof)
        assert normwise(op.apply(dev(x)).cpu().numpy(), P.apply(x)) <= PARITY_TOL


@pytest.mark.parametrize("kind,n,p", [("diffusion", (12, 12, 12), 4), ("diffusion", (6, 6, 6), 8),
                                      ("mass", (20, 20, 20), 2), ("diffusion", (40, 8, 10), 3)])
def test_apply_medium_meshes(kind, n, p):
    op = make(kind, n, p)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(0).standard_normal(P.ndof)
    assert normwise(op.apply(dev(x)).cpu().numpy(), P.apply(x)) <= PARITY_TOL


def test_apply_full_bp3_p4_config():
    """BASELINE configs[1]: BP3 p=4 on 54^3 (10.2 M dofs) — direct parity with the
    oracle plus size-independent properties (symmetry, null space, linearity)."""
    op = make("diffusion", (54, 54, 54), 4)
    assert op.num_dofs == 10218313
    rng = np.random.default_rng(0)
    x = rng.standard_normal(op.num_dofs)
    xd = dev(x)
    y = op.apply(xd)
    P = bp.Problem("diffusion", 54, 54, 54, 4)
    assert normwise(y.cpu().numpy(), P.apply(x, chunk=16384)) <= PARITY_TOL
    z = dev(rng.standard_normal(op.num_dofs))
    Az = op.apply(z)
    s1, s2 = float(torch.dot(z, y)), float(torch.dot(xd, Az))
    assert abs(s1 - s2) <= 1e-12 * (abs(s1) + float(torch.linalg.vector_norm(y) * torch.linalg.vector_norm(z)) * 1e-3)
    ones = torch.ones_like(xd)
    assert float(op.apply(ones).abs().max()) <= 1e-12 * float(y.abs().max())
    lin = op.apply(2.0 * xd - 3.0 * z)
    assert float((lin - (2.0 * y - 3.0 * Az)).abs().max()) <= 1e-12 * float(lin.abs().max())


def test_host_buffers_match_device_path(golden):
    op = make("diffusion", (3, 3, 3), 4)
    x = golden["bp3_3x3x3_p4_x"]
    yh = op.apply(x)
    assert isinstance(yh, np.ndarray)
    assert normwise(yh, op.apply(dev(x)).cpu().numpy()) <= 1e-15
    assert normwise(yh, golden["bp3_3x3x3_p4_y"]) <= PARITY_TOL


@pytest.mark.parametrize("kind,n,p", [("diffusion", (5, 4, 9), 3), ("mass", (3, 3, 17), 5),
                                      ("diffusion", (6, 5, 4), 8)])
def test_host_buffers_chunk_pipeline(kind, n, p):
    """fk_op_apply_host splits nz >= 4 meshes into z-chunks (H2D / compute /
    D2H overlapped); each plane must still receive every element's share."""
    import torch as _t

    op = make(kind, n, p)
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(5).standard_normal(P.ndof)
    xh = _t.from_numpy(x).pin_memory().numpy()
    yh = _t.empty(P.ndof, dtype=_t.float64).pin_memory().numpy()
    op.apply_host(xh, yh)
    assert normwise(yh, P.apply(x)) <= PARITY_TOL
    # pageable buffers take the same path
    assert normwise(op.apply(x), P.apply(x)) <= PARITY_TOL


@pytest.mark.parametrize("kind,n,p,world", [("diffusion", (4, 3, 7), 3, 3), ("mass", (3, 3, 4), 5, 2),
                                             ("diffusion", (5, 5, 8), 4, 4)])
@pytest.mark.parametrize("dirichlet", [False, True])
def test_zslab_loopback_matches_single_gpu(kind, n, p, world, dirichlet):
    """The multi-GPU decomposition on one device: every rank's z-slab operator
    (local restriction offsets, slab Dirichlet faces) applied element-locally,
    interface planes summed by hand (what fk_comm.cu does over NCCL), then the
    Dirichlet copy — must equal the single-GPU / oracle apply."""
    from paper_2603_09038_b200 import parallel

    nx, ny, nz = n
    P = bp.Problem(kind, *n, p)
    x = np.random.default_rng(11).standard_normal(P.ndof)
    ref = P.constrained_apply(x, P.boundary()) if dirichlet else P.apply(x)
    plane = parallel.plane_size(nx, ny, p)
    parts = []
    for r in range(world):
        z0, z1 = parallel.slab_range(nz, r, world)
        op = make(kind, n, p, z_range=(z0, z1), dirichlet=dirichlet)
        s, e = parallel.local_dof_range(nx, ny, p, z0, z1)
        assert op.dof_offset == s and op.num_dofs == e - s
        assert np.array_equal(op.restriction_ids(), bp.gather_ids(nx, ny, nz, p + 1, (z0, z1)))
        xl = dev(x[s:e])
        if dirichlet:
            xl = op.set_essential(xl.clone(), 0.0)
        parts.append((op, s, e, op.apply_local(xl).cpu().numpy()))
    y = np.zeros(P.ndof)
    for op, s, e, yl in parts:
        y[s:e] += yl  # shared planes receive both partial sums
    if dirichlet:
        ess = P.boundary()
        y[ess] = x[ess]
    assert normwise(y, ref) <= PARITY_TOL


def test_comm_single_rank_path():
    """fk_comm_create through the dlopen'ed NCCL (the copy torch loaded) with one
    rank: exchange and allreduce are no-ops, results unchanged."""
    import torch.distributed as dist

    from paper_2603_09038_b200 import Comm

    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29577", rank=0, world_size=1)
    comm = Comm(0, 1, 0)
    op = make("diffusion", (3, 3, 4), 3, dirichlet=True, comm=comm)
    ref = make("diffusion", (3, 3, 4), 3, dirichlet=True)
    x = dev(np.random.default_rng(2).standard_normal(op.num_dofs))
    assert normwise(op.apply(x).cpu().numpy(), ref.apply(x).cpu().numpy()) <= 1e-15
    b = ref.set_essential(dev(np.random.default_rng(3).standard_normal(op.num_dofs)), 0.0)
    _, h1 = cg_solve(op, b, iters=30)
    _, h2 = cg_solve(ref, b, iters=30)
    assert np.max(np.abs(h1 - h2)) <= 1e-10 * h2[0]
    op.close()
    comm.close()
    dist.destroy_process_group()


def test_mass_integrates_volume():
    for ext in ((1.0, 1.0, 1.0), (2.0, 1.0, 0.5)):
        op = make("mass", (4, 3, 5), 5, ext=ext)
        one = torch.ones(op.num_dofs, dtype=torch.float64, device="cuda")
        assert abs(float(torch.dot(one, op.apply(one))) - ext[0] * ext[1] * ext[2]) < 1e-13


# -- diagonal, Dirichlet, CG ----------------------------------------------------------


@pytest.mark.parametrize("key,kind,n,p,q,ext", [
    ("bp1_8x8x8_p2", "mass", (8, 8, 8), 2, None, (1.0, 1.0, 1.0)),
    ("bp3_3x3x3_p4", "diffusion", (3, 3, 3), 4, None, (1.0, 1.0, 1.0)),
    ("bp3_3x3x3_p8", "diffusion", (3, 3, 3), 8, None, (1.0, 1.0, 1.0)),
    ("bp3_2x3x2_p3_aniso", "diffusion", (2, 3, 2), 3, None, (2.0, 1.0, 0.5)),
])
def test_diagonal_matches_reference(golden, key, kind, n, p, q, ext):
    op = make(kind, n, p, q, ext)
    assert normwise(op.diagonal().cpu().numpy(), golden[key + "_diag"]) <= PARITY_TOL


@pytest.mark.parametrize("p", [2, 4, 6])
def test_dirichlet_constrained_apply(p):
    n = (3, 4, 2)
    op = make("diffusion", n, p, dirichlet=True)
    P = bp.Problem("diffusion", *n, p)
    ess = P.boundary()
    x = np.random.default_rng(3).standard_normal(P.ndof)
    assert normwise(op.apply(dev(x)).cpu().numpy(), P.constrained_apply(x, ess)) <= PARITY_TOL
    d = P.diagonal()
    d[ess] = 1.0
    assert normwise(op.diagonal().cpu().numpy(), d) <= PARITY_TOL


@pytest.mark.parametrize("key,n,p", [("cg_3x3x3_p3", (3, 3, 3), 3), ("cg_2x2x3_p5", (2, 2, 3), 5)])
def test_cg_history_matches_reference(golden, key, n, p):
    op = make("diffusion", n, p, dirichlet=True)
    href = golden[key + "_hist"]
    x, hist = cg_solve(op, golden[key + "_b"], iters=len(href) - 1)
    assert len(hist) == len(href)
    assert np.max(np.abs(hist - href)) <= 1e-8 * href[0]
    assert normwise(x, golden[key + "_x"]) <= 1e-8


def test_cg_100_iterations_vs_oracle():
    n, p = (6, 5, 7), 4
    op = make("diffusion", n, p, dirichlet=True)
    P = bp.Problem("diffusion", *n, p)
    b = np.random.default_rng(0).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    xr, hr = P.pcg(b, iters=100)
    x, h = cg_solve(op, dev(b), iters=100)
    assert len(h) == 101
    assert np.max(np.abs(h - hr)) <= 1e-8 * hr[0]
    assert normwise(x.cpu().numpy(), xr) <= 1e-8


def test_cg_rtol_stops_early():
    op = make("diffusion", (4, 4, 4), 3, dirichlet=True)
    b = np.random.default_rng(1).standard_normal(op.num_dofs)
    b[fem.boundary_dofs(4, 4, 4, 4)] = 0.0
    P = bp.Problem("diffusion", 4, 4, 4, 3)
    _, hr = P.pcg(b, iters=200, rtol=1e-6)
    _, h = cg_solve(op, b, iters=200, rtol=1e-6)
    assert len(h) == len(hr) < 200
    assert h[-1] <= 1e-6 * h[0]


# -- API behaviour ------------------------------------------------------------------


def test_shape_errors_and_counters():
    op = make("diffusion", (2, 2, 2), 3)
    with pytest.raises(ValueError, match="do not match"):
        op.apply(torch.zeros(op.num_dofs + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="do not match"):
        op.apply(np.zeros(3))
    with pytest.raises(ValueError):
        make("diffusion", (2, 2, 2), 3, strategy="scalar")
    with pytest.raises(ValueError):  # MF runs the matrix-free variant only
        make("diffusion", (2, 2, 2), 3, strategy="MF", variant="dmma")
    with pytest.raises(NotImplementedError):
        make("diffusion", (2, 2, 2), 3, 9)
    before = op.counters.operator_applies
    op.apply(op.zeros())
    assert op.counters.operator_applies == before + 1
    assert op.counters.flops == op.flops_per_apply * op.counters.operator_applies


@pytest.mark.parametrize("strategy", ["MF", "FusedMF"])
@pytest.mark.parametrize("kind", ["mass", "diffusion"])
def test_matrix_free_strategy_matches_pa(strategy, kind):
    """The reference's MF strategy (operator.py:280-286: factors recomputed per
    element instead of read) through PAOperator(strategy=...) -> variant "mf"
    with no PA data traffic; same operator as PA to rounding."""
    for p, n in ((2, (5, 4, 3)), (4, (6, 5, 7)), (7, (3, 3, 2))):
        P = bp.Problem(kind, *n, p)
        x = np.random.default_rng(p).standard_normal(P.ndof)
        op = make(kind, n, p, strategy=strategy)
        assert op.variant == "mf"
        assert op.bytes_per_apply == 16 * P.ndof + 4 * (p + 1) ** 3 * P.ids.shape[0]
        assert normwise(op.apply(dev(x)).cpu().numpy(), P.apply(x)) <= PARITY_TOL


@pytest.mark.parametrize("qoff", [1, 2])
@pytest.mark.parametrize("p", [1, 3, 5, 8])
def test_matrix_free_anisotropic(p, qoff):
    """MF on a non-cubic box (jinv differs per direction, D_ss = w|J| jinv_s^2)
    and with q = p+1 and p+2, with Dirichlet bits."""
    ext = (2.0, 1.0, 0.5)
    n = (4, 3, 2) if p <= 4 else (2, 3, 2)
    P = bp.Problem("diffusion", *n, p, p + qoff, extents=ext)
    x = np.random.default_rng(p).standard_normal(P.ndof)
    op = make("diffusion", n, p, p + qoff, ext, strategy="MF", dirichlet=True)
    ref = P.constrained_apply(x, P.boundary())
    assert normwise(op.apply(dev(x)).cpu().numpy(), ref) <= PARITY_TOL


def test_reference_objects_drop_in(golden):
    """The operator consumes duck-typed mesh/basis objects (feklab's or ours)."""
    class RefLikeMesh:
        nx, ny, nz = 3, 3, 3
        jacobian_diag = np.array([1 / 6, 1 / 6, 1 / 6])
        jacobian_det = float(np.prod(np.array([1 / 6, 1 / 6, 1 / 6])))
        num_elements = 27

    b = fem.Basis1D.nodal(5, 6)
    op = PAOperator(RefLikeMesh(), 4, basis=b)
    y = op.apply(dev(golden["bp3_3x3x3_p4_x"])).cpu().numpy()
    assert normwise(y, golden["bp3_3x3x3_p4_y"]) <= PARITY_TOL


@pytest.mark.parametrize("p,n,variant,iters", [
    (6, (3, 3, 3), "auto", 60),   # BASELINE configs[4] order
    (6, (2, 3, 4), "mf", 60),     # matrix-free operator, as bench.py --cg ... --variant mf
    (4, (3, 3, 3), "mf", 80),
    (8, (2, 2, 2), "auto", 40),
    (5, (3, 2, 3), "dmma", 40),   # a non-QF kernel: p.Ap by the dot pass
])
def test_cg_more_orders_and_variants(p, n, variant, iters):
    """CG on the fused iteration (p.Ap as the kernel's element quadratic form
    for EO / MF geometries, the dot pass otherwise) against the oracle PCG."""
    P = bp.Problem("diffusion", *n, p)
    op = make("diffusion", n, p, dirichlet=True, variant=variant)
    b = np.random.default_rng(p).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    x, h = cg_solve(op, b, iters=iters)
    xr, hr = P.pcg(b, iters=iters)
    assert len(h) == len(hr) and np.max(np.abs(h - hr)) <= 1e-8 * hr[0]
    assert normwise(x, xr) <= 1e-8
