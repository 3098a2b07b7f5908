"""Golden vectors of the reference's acoustic-gravity block operator.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mixed.py

Writes tests/golden/golden_mixed.npz by calling the REAL reference only:
``feklab.operator.BlockOperator`` (``apply`` with the PA and FusedPA
strategies, ``apply_fused_normal``, ``apply_mass_inverse``, the lumped mass
diagonals of ``setup_quad_data``) and ``rk4_step``
(/root/reference/pkg/src/feklab/operator.py:221-397, 506-531).  The GPU box
never runs this file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from feklab.mesh import build_mesh  # noqa: E402
from feklab.operator import BlockOperator, State, rk4_step  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_mixed.npz")

# name: (mesh n, extents, order_p, order_u, q, rho, bulk, coupling_scale)
CASES = {
    "m111": ((1, 1, 1), (1.0, 1.0, 1.0), 4, 3, 5, 1.0, 1.0, 1.0),
    "m222": ((2, 2, 2), (1.0, 1.0, 1.0), 4, 3, 5, 1.0, 1.0, 1.0),
    "m322_p2u1": ((3, 2, 2), (2.0, 1.0, 0.5), 2, 1, 3, 1.0, 1.0, 1.0),
    "m232_p3u2": ((2, 3, 2), (1.0, 1.0, 1.0), 3, 2, 4, 2.0, 3.0, 1.5),
    "m333_p6u5": ((3, 3, 3), (1.0, 1.0, 1.0), 6, 5, 7, 1.0, 1.0, 1.0),
    "m443": ((4, 4, 3), (1.0, 1.0, 1.0), 4, 3, 5, 1025.0, 1025.0 * 1500.0 ** 2, 1.0),
}


def main():
    out = {}
    for name, (n, ext, op_, ou, q, rho, bulk, cs) in CASES.items():
        mesh = build_mesh(*n, extents=ext)
        ops = {s: BlockOperator(mesh, order_p=op_, order_u=ou, num_quad_1d=q, strategy=s,
                                rho=rho, bulk_modulus=bulk, coupling_scale=cs)
               for s in ("PA", "FusedPA")}
        op = ops["PA"]
        rng = np.random.default_rng(sum(n) + op_)
        s = op.zero_state()
        s.u = rng.standard_normal(s.u.shape)
        s.p = rng.standard_normal(s.p.shape)
        out[f"{name}_u"] = s.u
        out[f"{name}_p"] = s.p
        for strat, o in ops.items():
            r = o.apply(s)
            out[f"{name}_{strat}_out_u"] = r.u
            out[f"{name}_{strat}_out_p"] = r.p
        out[f"{name}_fused_normal"] = ops["FusedPA"].apply_fused_normal(s.u)
        out[f"{name}_lump_u"] = op.quad.lump_u
        out[f"{name}_lump_p"] = op.quad.lump_p
        mi = op.apply_mass_inverse(s)
        out[f"{name}_minv_u"] = mi.u
        out[f"{name}_minv_p"] = mi.p
        out[f"{name}_gather"] = op.restriction.gather_ids
        st = State(s.u.copy(), s.p.copy())
        for k in range(2):
            st = rk4_step(st, 1e-3, ops["FusedPA"], step_index=k)
        out[f"{name}_rk4_u"] = st.u
        out[f"{name}_rk4_p"] = st.p
        out[f"{name}_meta"] = np.array([*n, *ext, op_, ou, q, rho, bulk, cs])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
