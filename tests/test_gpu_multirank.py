"""The multi-rank library path (z-slabs) executed for real.

Every test builds a group of nranks = 2..4 z-slab operators on ONE GPU and
drives each rank from its own host thread and CUDA stream through the C-ABI:

* in-process (loopback) groups: ``Comm.loopback`` — the peer-memory
  transport of fk_comm.cu with every rank's mailbox on this device, i.e. the
  same put / flag / add kernels and slot allreduce that run over NVLink on
  an 8-GPU box, including apply_overlapped (nz_local >= 3), the owned-dof
  dots, slab Dirichlet faces and the CUDA-graph-captured CG;
* two processes: ``Comm(transport="p2p")`` with the mailboxes mapped through
  CUDA IPC, bootstrapped over gloo — the path bench.py --gpus N takes.

Results are compared with the single-process CPU oracle on the same global
mesh (normwise 1e-12; CG: identical iteration counts, histories within
1e-8 h_0, as tests/test_gpu_parity.py) and shared planes must be
bit-identical on both neighbours.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from _util import PARITY_TOL, normwise
from oracle import bp
from paper_2603_09038_b200 import Comm, PAOperator, cg_solve, fem, parallel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


class Group:
    """nranks z-slab operators of one global mesh on a loopback group."""

    def __init__(self, kind, n, p, world, dirichlet=False, variant="auto", q=None):
        self.kind, self.n, self.p, self.world = kind, n, p, world
        nx, ny, nz = n
        self.plane = parallel.plane_size(nx, ny, p)
        self.comms = Comm.loopback(world, self.plane)
        self.streams = [torch.cuda.Stream() for _ in range(world)]
        mesh = fem.build_mesh(*n)
        self.ops, self.ranges = [], []
        for r in range(world):
            self.ops.append(PAOperator(mesh, p, q, kind=kind, dirichlet=dirichlet, comm=self.comms[r],
                                       stream=self.streams[r], variant=variant))
            z0, z1 = self.comms[r].slab(nz)
            self.ranges.append(parallel.local_dof_range(nx, ny, p, z0, z1))
        self.P = bp.Problem(kind, *n, p, q)

    def local(self, x):
        return [dev(x[s:e]) for s, e in self.ranges]

    def empty(self):
        return [torch.empty(e - s, dtype=torch.float64, device="cuda") for s, e in self.ranges]

    def run(self, fn):
        torch.cuda.synchronize()
        return parallel.run_ranks(fn, self.world, streams=self.streams)

    def assemble(self, parts):
        """Global vector from the owned parts; checks both copies of every
        shared plane are bitwise identical."""
        y = np.zeros(self.P.ndof)
        for r, ((s, e), v) in enumerate(zip(self.ranges, parts)):
            v = v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)
            if r > 0:
                prev = parts[r - 1]
                prev = prev.cpu().numpy() if hasattr(prev, "cpu") else np.asarray(prev)
                assert np.array_equal(prev[-self.plane:], v[:self.plane]), \
                    f"shared plane of ranks {r - 1}/{r} differs"
            y[s:e] = v
        return y

    def close(self):
        for op in self.ops:
            op.close()
        for c in self.comms:
            c.close()


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
def test_loopback_apply_matches_oracle(kind, n, p, world, dirichlet):
    g = Group(kind, n, p, world, dirichlet)
    x = np.random.default_rng(7).standard_normal(g.P.ndof)
    ess = g.P.boundary()
    if dirichlet:
        x[ess] = 0.0
    ref = g.P.constrained_apply(x, ess) if dirichlet else g.P.apply(x)
    xs, ys = g.local(x), g.empty()

    def fn(r, s, bar):
        for _ in range(3):  # repeated exchanges: the flag sequence advances
            g.ops[r].apply(xs[r], out=ys[r])

    g.run(fn)
    y = g.assemble(ys)
    assert normwise(y, ref) <= PARITY_TOL
    g.close()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_loopback_dot_owned_dofs(world):
    g = Group("diffusion", (3, 2, 8), 3, world)
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(g.P.ndof), rng.standard_normal(g.P.ndof)
    xa, xb = g.local(a), g.local(b)
    vals = g.run(lambda r, s, bar: [g.ops[r].dot(xa[r], xb[r]) for _ in range(4)])
    ref = float(a @ b)
    for v in vals:
        # every rank holds the same bits (slot sums in rank order)
        assert v == vals[0]
        assert abs(v[0] - ref) <= 1e-13 * np.sqrt(float(a @ a) * float(b @ b))
    g.close()


@pytest.mark.parametrize("kind,n,p,world", [("diffusion", (3, 2, 6), 4, 3), ("mass", (2, 3, 4), 3, 2)])
def test_loopback_diagonal(kind, n, p, world):
    g = Group(kind, n, p, world, dirichlet=True)
    outs = g.empty()
    g.run(lambda r, s, bar: g.ops[r].diagonal(out=outs[r]))
    ref = g.P.diagonal()
    ref[g.P.boundary()] = 1.0
    assert normwise(g.assemble(outs), ref) <= PARITY_TOL
    g.close()


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
def test_loopback_cg_matches_oracle(kind, n, p, world, variant, iters):
    g = Group(kind, n, p, world, dirichlet=True, variant=variant)
    b = np.random.default_rng(0).standard_normal(g.P.ndof)
    b[g.P.boundary()] = 0.0
    bs, xs = g.local(b), g.empty()
    res = g.run(lambda r, s, bar: cg_solve(g.ops[r], bs[r], iters=iters, out=xs[r], barrier=bar)[1])
    xr, hr = g.P.pcg(b, iters=iters)
    for h in res:
        assert len(h) == len(hr)
        assert np.array_equal(h, res[0])  # identical scalars on every rank
        assert np.max(np.abs(h - hr)) <= 1e-8 * hr[0]
    x = g.assemble(xs)
    assert normwise(x, xr) <= 1e-8
    for op in g.ops:
        assert op.counters.operator_applies == iters
    g.close()


def test_loopback_cg_rtol_stops_every_rank_together():
    g = Group("diffusion", (3, 3, 6), 3, 3, dirichlet=True)
    b = np.random.default_rng(1).standard_normal(g.P.ndof)
    b[g.P.boundary()] = 0.0
    bs, xs = g.local(b), g.empty()
    res = g.run(lambda r, s, bar: cg_solve(g.ops[r], bs[r], iters=200, rtol=1e-6, out=xs[r],
                                           barrier=bar)[1])
    _, hr = g.P.pcg(b, iters=200, rtol=1e-6)
    assert all(len(h) == len(hr) for h in res) and len(hr) < 201
    g.close()


def test_loopback_matches_single_gpu_bitwise_inside_slabs():
    """Interior dofs of a slab see exactly the same element contributions in
    the same kernel as the single-GPU apply; only shared planes add two
    partial sums in a different order."""
    n, p = (3, 3, 8), 4
    g = Group("diffusion", n, p, 2)
    single = PAOperator(fem.build_mesh(*n), p)
    x = np.random.default_rng(9).standard_normal(g.P.ndof)
    ref = single.apply(dev(x)).cpu().numpy()
    xs, ys = g.local(x), g.empty()
    g.run(lambda r, s, bar: g.ops[r].apply(xs[r], out=ys[r]))
    y = g.assemble(ys)
    assert normwise(y, ref) <= 1e-15
    single.close()
    g.close()


def test_plane_capacity_is_checked():
    comms = Comm.loopback(2, 10)
    with pytest.raises(ValueError, match="do(es)? not match"):
        PAOperator(fem.build_mesh(3, 3, 4), 3, comm=comms[0])
    for c in comms:
        c.close()


# -- two processes, CUDA IPC mailboxes -------------------------------------------------

WORKER = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["FK_ROOT"]); sys.path.insert(0, os.path.join(os.environ["FK_ROOT"], "tests"))
from paper_2603_09038_b200 import Comm, PAOperator, cg_solve, fem, parallel
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["FK_PORT"], rank=rank, world_size=world)
torch.cuda.set_device(0)
n, p = (3, 2, 6), 4
comm = Comm(rank, world, 0, transport="p2p")
s = torch.cuda.Stream()
op = PAOperator(fem.build_mesh(*n), p, dirichlet=True, comm=comm, stream=s)
z0, z1 = comm.slab(n[2])
lo, hi = parallel.local_dof_range(n[0], n[1], p, z0, z1)
rng = np.random.default_rng(0)
x = rng.standard_normal((n[0]*p+1)*(n[1]*p+1)*(n[2]*p+1))
with torch.cuda.stream(s):
    xl = torch.as_tensor(x[lo:hi], device="cuda")
    y = op.apply(xl)
    b = op.set_essential(xl.clone(), 0.0)
    xs, h = cg_solve(op, b, iters=25)
    d = op.dot(xl, xl)
s.synchronize()
np.savez(os.environ["FK_OUT"] + f"_{rank}.npz", y=y.cpu().numpy(), x=xs.cpu().numpy(), h=h, d=d, lo=lo, hi=hi)
dist.barrier()
op.close(); comm.close()
dist.destroy_process_group()
"""


def test_two_process_ipc_p2p(tmp_path):
    n, p, world = (3, 2, 6), 4, 2
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = str(29600 + os.getpid() % 300)
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), FK_ROOT=ROOT, FK_PORT=port,
                   FK_OUT=str(tmp_path / "out"))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    for pr in procs:
        out, _ = pr.communicate(timeout=300)
        assert pr.returncode == 0, out.decode()[-3000:]
    P = bp.Problem("diffusion", *n, p)
    x = np.random.default_rng(0).standard_normal(P.ndof)
    ess = P.boundary()
    res = [np.load(tmp_path / f"out_{r}.npz") for r in range(world)]
    y = np.zeros(P.ndof)
    xs = np.zeros(P.ndof)
    for r in res:
        y[int(r["lo"]):int(r["hi"])] = r["y"]
        xs[int(r["lo"]):int(r["hi"])] = r["x"]
    plane = parallel.plane_size(n[0], n[1], p)
    assert np.array_equal(res[0]["y"][-plane:], res[1]["y"][:plane])
    assert normwise(y, P.constrained_apply(x, ess)) <= PARITY_TOL
    b = x.copy()
    b[ess] = 0.0
    xr, hr = P.pcg(b, iters=25)
    for r in res:
        assert len(r["h"]) == len(hr) and np.max(np.abs(r["h"] - hr)) <= 1e-8 * hr[0]
        assert abs(float(r["d"]) - float(x @ x)) <= 1e-12 * float(x @ x)
    assert normwise(xs, xr) <= 1e-8
