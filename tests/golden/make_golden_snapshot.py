"""Reference snapshot file (feklab.solver.save_snapshot, solver.py:179-198)
for the wire-format test.  Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_snapshot.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from feklab.mesh import build_mesh  # noqa: E402
from feklab.operator import BlockOperator  # noqa: E402
from feklab.solver import save_snapshot  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "snapshot_ref.bin")

mesh = build_mesh(2, 1, 2, extents=(2.0, 1.0, 0.5))
op = BlockOperator(mesh, order_p=2, order_u=1, num_quad_1d=3)
s = op.zero_state()
rng = np.random.default_rng(3)
s.u = rng.standard_normal(s.u.shape)
s.p = rng.standard_normal(s.p.shape)
save_snapshot(OUT, s, mesh)
print("wrote", OUT, os.path.getsize(OUT), "bytes")
