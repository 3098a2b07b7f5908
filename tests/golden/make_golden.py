"""Generate golden vectors by importing the REAL reference (feklab).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Everything here calls reference functions
only (Basis1D.nodal, build_mesh, h1_restriction, _quad_weights_3d,
apply_basis_3d / apply_basis_transpose_3d / apply_gradient_3d /
apply_gradient_transpose_3d, Restriction.gather / scatter_add), composed per
SURVEY.md §8c.  CG and the Jacobi diagonal are not in the reference; they
are composed here from the same reference calls (MFEM CGSolver semantics).
The GPU box never runs this file (it has no /root/reference).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from feklab.mesh import build_mesh, h1_restriction, h1_node_coords  # noqa: E402
from feklab.operator import _quad_weights_3d  # noqa: E402
from feklab.tensor import (  # noqa: E402
    Basis1D,
    Tensor3,
    apply_basis_3d,
    apply_basis_transpose_3d,
    apply_gradient_3d,
    apply_gradient_transpose_3d,
)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def setup(n, p, q=None, extents=(1.0, 1.0, 1.0)):
    nx, ny, nz = n
    mesh = build_mesh(nx, ny, nz, extents)
    q = p + 2 if q is None else q
    b = Basis1D.nodal(p + 1, q)
    r = h1_restriction(mesh, p + 1)
    wdet = _quad_weights_3d(b) * mesh.jacobian_det
    jinv = 1.0 / mesh.jacobian_diag
    return mesh, b, r, wdet, jinv


def ref_apply(kind, b, r, wdet, jinv, x):
    d, q = b.num_dofs_1d, b.num_quad_1d
    xe = r.gather(x)
    ye = np.empty_like(xe)
    for e in range(xe.shape[0]):
        X = Tensor3((d, d, d), xe[e].copy())
        if kind == "mass":
            u = apply_basis_3d(b, X)
            ye[e] = apply_basis_transpose_3d(b, Tensor3((q, q, q), wdet * u.data)).data
        else:
            g = apply_gradient_3d(b, X)
            t = tuple(Tensor3((q, q, q), wdet * jinv[s] ** 2 * g[s].data) for s in range(3))
            ye[e] = apply_gradient_transpose_3d(b, t).data
    return r.scatter_add(ye)


def ref_diagonal(kind, b, r, wdet, jinv):
    d, q = b.num_dofs_1d, b.num_quad_1d
    b2 = Basis1D(d, q, b.values ** 2, b.gradients ** 2)
    if kind == "mass":
        de = apply_basis_transpose_3d(b2, Tensor3((q, q, q), wdet.copy())).data
    else:
        t = tuple(Tensor3((q, q, q), wdet * jinv[s] ** 2) for s in range(3))
        de = apply_gradient_transpose_3d(b2, t).data
    nel = r.gather_ids.shape[0]
    return r.scatter_add(np.broadcast_to(de, (nel, de.size)).copy())


def boundary_ids(mesh, p):
    npx, npy, npz = mesh.nx * p + 1, mesh.ny * p + 1, mesh.nz * p + 1
    gk, gj, gi = np.meshgrid(np.arange(npz), np.arange(npy), np.arange(npx), indexing="ij")
    on = (gi == 0) | (gi == npx - 1) | (gj == 0) | (gj == npy - 1) | (gk == 0) | (gk == npz - 1)
    return np.flatnonzero(on.ravel())


def ref_pcg(b_vec, apply, diag, ess, iters):
    dinv = 1.0 / diag
    dinv[ess] = 1.0

    def A(v):
        vz = v.copy()
        vz[ess] = 0.0
        y = apply(vz)
        y[ess] = v[ess]
        return y

    x = np.zeros_like(b_vec)
    rr = b_vec.copy()
    z = dinv * rr
    pp = z.copy()
    nom = float(rr @ z)
    hist = [np.sqrt(nom)]
    for _ in range(iters):
        Ap = A(pp)
        alpha = nom / float(pp @ Ap)
        x += alpha * pp
        rr -= alpha * Ap
        z = dinv * rr
        betanom = float(rr @ z)
        hist.append(np.sqrt(betanom))
        pp = z + (betanom / nom) * pp
        nom = betanom
    return x, np.array(hist)


def main():
    g = {}
    # 1D tables, d = 2..9, q = d+1 (p+2) and q = d (p+1)
    for d in range(2, 10):
        for q in (d + 1, d):
            b = Basis1D.nodal(d, q)
            g[f"basis_d{d}_q{q}_B"] = b.values
            g[f"basis_d{d}_q{q}_G"] = b.gradients
            g[f"basis_d{d}_q{q}_w"] = b.quad_weights
            g[f"basis_d{d}_q{q}_nodes"] = b.nodes
    # restriction maps (int64, bit-exact)
    for (n, d) in [((2, 3, 4), 3), ((3, 3, 3), 5), ((4, 2, 3), 2), ((2, 2, 2), 9)]:
        mesh = build_mesh(*n)
        r = h1_restriction(mesh, d)
        key = f"restr_{n[0]}x{n[1]}x{n[2]}_d{d}"
        g[key] = r.gather_ids
        g[key + "_mult"] = r.multiplicity()
    # node coordinates
    mesh = build_mesh(2, 3, 2, (2.0, 1.0, 0.5))
    g["coords_2x3x2_d4"] = h1_node_coords(mesh, Basis1D.nodal(4, 5).nodes)

    cases = [("mass", (8, 8, 8), 2, None, (1.0, 1.0, 1.0), "bp1_8x8x8_p2")]
    for p in range(1, 9):
        cases.append(("diffusion", (3, 3, 3), p, None, (1.0, 1.0, 1.0), f"bp3_3x3x3_p{p}"))
        cases.append(("mass", (2, 2, 2), p, None, (1.0, 1.0, 1.0), f"bp1_2x2x2_p{p}"))
    cases.append(("diffusion", (2, 3, 2), 3, None, (2.0, 1.0, 0.5), "bp3_2x3x2_p3_aniso"))
    cases.append(("diffusion", (3, 2, 4), 4, 5, (1.0, 1.0, 1.0), "bp3_3x2x4_p4_q5"))
    cases.append(("mass", (3, 2, 4), 4, 5, (1.0, 1.5, 1.0), "bp1_3x2x4_p4_q5"))
    for kind, n, p, q, ext, key in cases:
        mesh, b, r, wdet, jinv = setup(n, p, q, ext)
        x = np.random.default_rng(0).standard_normal(r.num_global)
        g[key + "_x"] = x
        g[key + "_y"] = ref_apply(kind, b, r, wdet, jinv, x)
        g[key + "_diag"] = ref_diagonal(kind, b, r, wdet, jinv)
        print(key, r.num_global, flush=True)

    # CG: BP3, Dirichlet on all faces, random b (seed 0) with boundary zeroed
    for n, p, iters in [((3, 3, 3), 3, 100), ((2, 2, 3), 5, 60)]:
        mesh, b, r, wdet, jinv = setup(n, p)
        ess = boundary_ids(mesh, p)
        rhs = np.random.default_rng(0).standard_normal(r.num_global)
        rhs[ess] = 0.0
        diag = ref_diagonal("diffusion", b, r, wdet, jinv)
        x, hist = ref_pcg(rhs, lambda v: ref_apply("diffusion", b, r, wdet, jinv, v), diag, ess, iters)
        key = f"cg_{n[0]}x{n[1]}x{n[2]}_p{p}"
        g[key + "_b"] = rhs
        g[key + "_x"] = x
        g[key + "_hist"] = hist
        print(key, hist[0], hist[-1], flush=True)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
