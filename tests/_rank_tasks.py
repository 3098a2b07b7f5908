"""Per-rank bodies of the multi-rank GPU tests (run inside tests/_rankpool.py
workers; one process per rank, all on cuda:0, P2P mailboxes over CUDA IPC).

Every task builds its z-slab communicator and operators from scratch, runs
through the public API (C-ABI underneath) and returns NumPy results with the
rank's global dof range; the parent assembles and checks them against the
oracle.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from paper_2603_09038_b200 import Comm, PAOperator, cg_solve, fem, parallel


def _ndof(n, p):
    return (n[0] * p + 1) * (n[1] * p + 1) * (n[2] * p + 1)


class _Slab:
    def __init__(self, rank, world, kind, n, p, transport="p2p", extents=(1.0, 1.0, 1.0), q=None, **kw):
        self.comm = Comm(rank, world, 0, transport=transport)
        self.stream = torch.cuda.Stream()
        self.op = PAOperator(fem.build_mesh(*n, extents=extents), p, q, kind=kind, comm=self.comm,
                             stream=self.stream, **kw)
        z0, z1 = self.comm.slab(n[2])
        self.lo, self.hi = parallel.local_dof_range(n[0], n[1], p, z0, z1)

    def local(self, x):
        with torch.cuda.stream(self.stream):
            t = torch.as_tensor(np.ascontiguousarray(x[self.lo:self.hi]), device="cuda")
        self.stream.synchronize()
        return t

    def close(self):
        torch.cuda.synchronize()
        dist.barrier()  # no rank unmaps its mailbox while a peer may still write to it
        self.op.close()
        self.comm.close()


def task_apply(rank, world, kind, n, p, dirichlet=False, seed=7, reps=3, variant="auto",
               deterministic=False, extents=(1.0, 1.0, 1.0), q=None):
    s = _Slab(rank, world, kind, n, p, dirichlet=dirichlet, variant=variant,
              deterministic=deterministic, extents=extents, q=q)
    x = np.random.default_rng(seed).standard_normal(_ndof(n, p))
    xl = s.local(x)
    ys = []
    with torch.cuda.stream(s.stream):
        y = torch.empty_like(xl)
        for _ in range(reps):  # repeated exchanges: the flag sequence advances
            s.op.apply(xl, out=y)
            ys.append(y.cpu().numpy())
    out = {"lo": s.lo, "hi": s.hi, "y": ys[-1], "all": ys, "variant": s.op.variant,
           "launch": s.op.launch}
    s.close()
    return out


def task_dot(rank, world, n, p, seed=3, reps=4):
    s = _Slab(rank, world, "diffusion", n, p)
    rng = np.random.default_rng(seed)
    a, b = rng.standard_normal(_ndof(n, p)), rng.standard_normal(_ndof(n, p))
    al, bl = s.local(a), s.local(b)
    with torch.cuda.stream(s.stream):
        vals = [s.op.dot(al, bl) for _ in range(reps)]
    s.close()
    return vals


def task_diagonal(rank, world, kind, n, p, deterministic=False):
    s = _Slab(rank, world, kind, n, p, dirichlet=True, deterministic=deterministic)
    with torch.cuda.stream(s.stream):
        d = s.op.diagonal().cpu().numpy()
    out = {"lo": s.lo, "hi": s.hi, "d": d}
    s.close()
    return out


def task_cg(rank, world, kind, n, p, iters, variant="auto", rtol=0.0, seed=0,
            deterministic=False, transport="p2p"):
    s = _Slab(rank, world, kind, n, p, dirichlet=True, variant=variant,
              deterministic=deterministic, transport=transport)
    from oracle import bp

    P = bp.Problem(kind, *n, p)
    b = np.random.default_rng(seed).standard_normal(P.ndof)
    b[P.boundary()] = 0.0
    bl = s.local(b)
    with torch.cuda.stream(s.stream):
        x, h = cg_solve(s.op, bl, iters=iters, rtol=rtol)
        x = x.cpu().numpy()
    out = {"lo": s.lo, "hi": s.hi, "x": x, "h": h, "applies": s.op.counters.operator_applies,
           "launch": s.op.launch}
    s.close()
    return out
