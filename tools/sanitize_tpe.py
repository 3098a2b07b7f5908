"""compute-sanitizer workload for the thread-per-element BP1 kernel (cfgs 58-59, p = 1-2,
ragged groups, Dirichlet bits, several groups per warp via FK_MAX_BLOCKS=2)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("FK_MAX_BLOCKS", "2")
from paper_2603_09038_b200 import PAOperator, build_mesh
torch.cuda.set_device(0)
for p in (1, 2):
    for cfg in (58, 59):
        for n in ((3, 2, 3), (7, 5, 3)):
            for dirichlet in (False, True):
                op = PAOperator(build_mesh(*n), p, kind="mass", dirichlet=dirichlet)
                op.set_config("eo", cfg)
                y = op.apply(torch.randn(op.num_dofs, dtype=torch.float64, device="cuda"))
                assert bool(torch.isfinite(y).all())
                op.close()
torch.cuda.synchronize(); print("tpe sanitize workload done")
