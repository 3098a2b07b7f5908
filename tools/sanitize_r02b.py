"""compute-sanitizer workload for the late round-2 kernels: the staged
scatter (EO cfgs 40-49, incl. PA data in registers), stages B-D fused in
registers (cfgs 50-53), the PA data streamed through a ring of c-plane pairs
(cfgs 54-57, mbarrier ring with cross-batch prefetch: FK_MAX_BLOCKS=2 makes
every CTA walk several batches) and the block operator's staged outputs
(mixed cfgs 4-7) and its single-X twins (mixed cfgs 8-15, several batches per CTA).

    compute-sanitizer --tool memcheck  python tools/sanitize_r02b.py
    compute-sanitizer --tool racecheck python tools/sanitize_r02b.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FK_MAX_BLOCKS", "2")

from paper_2603_09038_b200 import MixedOperator, MixedState, PAOperator, build_mesh  # noqa: E402

torch.cuda.set_device(0)


def finite(t):
    assert bool(torch.isfinite(torch.as_tensor(t)).all())


for p, cfgs, kind in ((3, range(40, 54), "mass"), (4, range(40, 58), "diffusion"), (5, range(54, 58), "diffusion"),
                      (4, range(40, 54), "mass")):
    for cfg in cfgs:
        for dirichlet in (False, True):
            op = PAOperator(build_mesh(3, 2, 3), p, kind=kind, dirichlet=dirichlet)
            try:
                op.set_config("eo", cfg)
            except NotImplementedError:
                op.close()
                continue
            finite(op.apply(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")))
            op.close()
for cfg in range(4, 16):
    os.environ["FK_MIX_CFG"] = str(cfg)
    for p in (3, 4):
        mop = MixedOperator(build_mesh(4, 3, 3), p, p - 1, p + 1)
        s = MixedState(torch.randn(mop.u_shape, dtype=torch.float64, device="cuda"),
                       torch.randn(mop.num_p, dtype=torch.float64, device="cuda"))
        r = mop.apply(s)
        finite(r.u)
        finite(r.p)
        mop.close()
torch.cuda.synchronize()
print("sanitize r02b workload done")
