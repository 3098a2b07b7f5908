"""Golden vectors of the reference block operator's boundary terms, forcing and counters.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mixed_bc.py

Writes tests/golden/golden_mixed_bc.npz by calling the REAL reference only
(/root/reference/pkg/src/feklab/operator.py):

* ``BlockOperator(absorbing=True).apply``         impedance pairing on the
  lateral faces (:357-358, _apply_absorbing :432-439)
* ``BlockOperator(surface_gravity=g)``            free-surface lumped mass
  (:268-276) -> ``quad.lump_p``, ``apply_mass_inverse``, ``surface_height``
* ``bottom_face_load(profile)``                   (:441-460)
* ``rk4_step(..., forcing=f, t=t0)``              forced RK4 (:506-531)
* ``counters`` after apply / apply_fused_normal   (:280-286, counters.py)

The GPU box never runs this file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from feklab.counters import Counters  # noqa: E402
from feklab.mesh import build_mesh  # noqa: E402
from feklab.operator import BlockOperator, State, rk4_step  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_mixed_bc.npz")

# name: (mesh n, extents, order_p, order_u, q, rho, bulk, coupling_scale, gravity)
CASES = {
    "b222": ((2, 2, 2), (1.0, 1.0, 1.0), 4, 3, 5, 1.0, 1.0, 1.0, 9.81),
    "b322_p2": ((3, 2, 2), (2.0, 1.0, 0.5), 2, 1, 3, 1.3, 2.0, 1.0, 2.0),
    "b232_p3cs": ((2, 3, 2), (1.0, 1.0, 1.0), 3, 2, 4, 2.0, 3.0, 1.5, 5.0),
    "b333_p6": ((3, 3, 3), (1.0, 1.0, 1.0), 6, 5, 7, 1.0, 1.0, 1.0, 1.0),
}


def profile(x, y):
    return np.sin(np.pi * x) * np.cos(0.5 * y) + 0.25 * x * y


def main():
    out = {}
    for name, (n, ext, op_, ou, q, rho, bulk, cs, g) in CASES.items():
        mesh = build_mesh(*n, extents=ext)
        nel = mesh.num_elements
        # per-element material (exercises the element-wise impedance / surface terms)
        rho_e = rho * (1.0 + 0.1 * np.arange(nel) / nel)
        bulk_e = bulk * (1.0 + 0.05 * np.cos(np.arange(nel)))
        kw = dict(order_p=op_, order_u=ou, num_quad_1d=q, rho=rho_e, bulk_modulus=bulk_e,
                  coupling_scale=cs)
        absorb = BlockOperator(mesh, strategy="FusedPA", absorbing=True, **kw)
        surf = BlockOperator(mesh, strategy="FusedPA", surface_gravity=g, **kw)
        both = BlockOperator(mesh, strategy="FusedPA", absorbing=True, surface_gravity=g, **kw)
        rng = np.random.default_rng(sum(n) + 7 * op_)
        s = absorb.zero_state()
        s.u = rng.standard_normal(s.u.shape)
        s.p = rng.standard_normal(s.p.shape)
        out[f"{name}_u"], out[f"{name}_p"] = s.u, s.p
        out[f"{name}_rho"], out[f"{name}_bulk"] = rho_e, bulk_e
        r = absorb.apply(s)
        out[f"{name}_absorb_out_u"], out[f"{name}_absorb_out_p"] = r.u, r.p
        out[f"{name}_surf_lump_p"] = surf.quad.lump_p
        mi = surf.apply_mass_inverse(s)
        out[f"{name}_surf_minv_p"] = mi.p
        out[f"{name}_surf_height"] = surf.surface_height(s)
        out[f"{name}_bottom_load"] = absorb.bottom_face_load(profile)

        def forcing(t, _s=s):
            f = both.zero_state()
            f.u = np.sin(3.0 * t) * _s.u[::-1].copy()
            f.p = np.cos(2.0 * t) * np.linspace(-1.0, 1.0, f.p.size)
            return f

        st = State(s.u.copy(), s.p.copy())
        t0 = 0.25
        for k in range(2):
            st = rk4_step(st, 2e-3, both, forcing=forcing, t=t0 + k * 2e-3, step_index=k)
        out[f"{name}_rk4f_u"], out[f"{name}_rk4f_p"] = st.u, st.p
        # counters (counters.py; _dfactors :280-286)
        for strat in ("PA", "FusedPA", "MF", "FusedMF"):
            c = Counters()
            o = BlockOperator(mesh, strategy=strat, counters=c, **kw)
            o.apply(s)
            a = (c.operator_applies, c.flops, c.d_reads)
            c.reset()
            o.apply_fused_normal(s.u)
            out[f"{name}_counters_{strat}"] = np.array([*a, c.operator_applies, c.flops, c.d_reads],
                                                       dtype=np.int64)
        out[f"{name}_meta"] = np.array([*n, *ext, op_, ou, q, rho, bulk, cs, g])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
