"""compute-sanitizer workload for the kernels added in round 2:
the quadratic-form CG geometries (QF twins, PA and MF, p = 2..8), the
deterministic colour mode (apply, diagonal, CG), the closed-form box
diagonal, the paper-style map DMMA body (p = 3, cfgs 3-5) and the new DMMA
geometries (cfgs 6-8), the warp-per-element and hybrid bodies (cfgs 9-14), the block operator's absorbing faces / free surface /
bottom load / forced RK4, and a single-rank P2P communicator (its exchange
kernels early-return; the multi-rank protocol runs in the rank-process tests).

    compute-sanitizer --tool memcheck python tools/sanitize_r02.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_09038_b200 import (Comm, MixedOperator, MixedState, PAOperator, build_mesh,  # noqa: E402
                                   cg_solve, rk4_step)

torch.cuda.set_device(0)


def finite(t):
    assert bool(torch.isfinite(torch.as_tensor(t)).all())


for p in range(2, 9):
    for strategy in ("PA", "MF"):
        op = PAOperator(build_mesh(3, 2, 3), p, dirichlet=True, strategy=strategy)
        b = op.set_essential(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda"), 0.0)
        x, h = cg_solve(op, b, iters=4)
        finite(x)
        op.close()
for p in (2, 4, 7):
    op = PAOperator(build_mesh(3, 3, 2), p, dirichlet=True, deterministic=True)
    x = torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")
    finite(op.apply(x))
    finite(op.diagonal())
    finite(cg_solve(op, op.set_essential(x.clone(), 0.0), iters=3)[0])
    op.close()
for kind in ("mass", "diffusion"):
    op = PAOperator(build_mesh(4, 3, 2), 5, kind=kind)
    finite(op.diagonal())
    op.close()
for cfg in range(3, 15):
    for kind in ("mass", "diffusion"):
        for dirichlet in (False, True):
            op = PAOperator(build_mesh(3, 2, 3), 3, kind=kind, dirichlet=dirichlet)
            op.set_config("dmma", cfg)
            finite(op.apply(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")))
            op.close()
for p in (2, 4, 6):
    mop = MixedOperator(build_mesh(2, 3, 2), p, p - 1, p + 1, absorbing=True, surface_gravity=9.8)
    s = MixedState(torch.randn(mop.u_shape, dtype=torch.float64, device="cuda"),
                   torch.randn(mop.num_p, dtype=torch.float64, device="cuda"))
    r = mop.apply(s)
    finite(r.u)
    finite(r.p)
    finite(mop.bottom_face_load(lambda x, y: np.sin(x) + y))
    f = lambda t: MixedState(torch.ones_like(s.u) * t, torch.ones_like(s.p))  # noqa: E731
    finite(rk4_step(s, 1e-3, mop, forcing=f, t=0.1).p)
    mop.close()
comm = Comm(0, 1, 0, transport="p2p", plane_cap=4096)
op = PAOperator(build_mesh(3, 3, 4), 3, dirichlet=True, comm=comm)
finite(op.apply(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")))
op.close()
comm.close()
torch.cuda.synchronize()
print("sanitize r02 workload done")
