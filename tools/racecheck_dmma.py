"""racecheck / synccheck workload for the shuffle- and shared-memory-heavy
DMMA bodies (warp-per-element cfgs 9-11, hybrid cfgs 12-14), p = 3:

    compute-sanitizer --tool racecheck --racecheck-report hazard python tools/racecheck_dmma.py
"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2603_09038_b200 import PAOperator, build_mesh
torch.cuda.set_device(0)
for cfg in range(9, 15):
    for kind in ("mass", "diffusion"):
        op = PAOperator(build_mesh(2, 2, 2), 3, kind=kind)
        op.set_config("dmma", cfg)
        y = op.apply(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda"))
        assert bool(torch.isfinite(y).all())
        op.close()
torch.cuda.synchronize(); print("racecheck workload done")
