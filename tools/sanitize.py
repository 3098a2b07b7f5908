"""Small applies for compute-sanitizer (memcheck / racecheck / synccheck):
every default geometry at p=1..8 (BP1, BP3, PA and MF, with Dirichlet bits),
the precomputed-gather / closed-form-id geometries (eo25-32, mf8-9) with and
without Dirichlet bits, the acoustic-gravity FusedPA/FusedMF apply and fused
normal at orders 2..8."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_09038_b200 import MixedOperator, MixedState, PAOperator, build_mesh

torch.cuda.set_device(0)
for p in range(1, 9):
    for kind in ("diffusion", "mass"):
        for strategy in ("PA", "MF"):
            op = PAOperator(build_mesh(3, 2, 2), p, kind=kind, strategy=strategy, dirichlet=(p % 2 == 0))
            x = torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")
            y = op.apply(x)
            assert bool(torch.isfinite(y).all())
            op.close()
for p in (1, 2, 4, 5, 8):
    for kind in ("diffusion", "mass"):
        for variant, cfgs in (("eo", range(25, 33)), ("mf", (8, 9))):
            for cfg in cfgs:
                for dirichlet in (False, True):
                    os.environ["FK_CFG"] = str(cfg)
                    op = PAOperator(build_mesh(3, 2, 2), p, kind=kind, dirichlet=dirichlet,
                                    strategy="MF" if variant == "mf" else "PA")
                    x = torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")
                    y = op.apply(x)
                    assert bool(torch.isfinite(y).all())
                    op.close()
os.environ.pop("FK_CFG", None)
for p in range(2, 9):
    for strategy in ("FusedPA", "FusedMF"):
        mop = MixedOperator(build_mesh(2, 2, 3), p, p - 1, p + 1, strategy=strategy)
        s = MixedState(torch.randn(mop.u_shape, dtype=torch.float64, device="cuda"),
                       torch.randn(mop.num_p, dtype=torch.float64, device="cuda"))
        r = mop.apply(s)
        assert bool(torch.isfinite(r.u).all()) and bool(torch.isfinite(r.p).all())
        mop.apply_fused_normal(s.u)
        mop.close()
torch.cuda.synchronize()
print("sanitize workload done")
