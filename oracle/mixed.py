"""NumPy restatement of the reference's acoustic-gravity block operator —
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference: /root/reference/pkg/src/feklab/operator.py
  * ``setup_quad_data``            :147-193  (dmat, wdet, lumped diagonals)
  * ``element_dfactors``           :137-144  (dm[q, s, s] = wdet * jinv_s)
  * ``BlockOperator.apply``        :331-362  (PA / FusedPA: the element loop
    order differs, the arithmetic per output entry does not)
  * ``_pressure_to_velocity``      :288-301  tau block
  * ``_velocity_to_pressure``      :303-319  v block, scattered with a minus
  * ``apply_fused_normal``         :364-387
  * ``apply_mass_inverse``         :391-397
  * ``rk4_step``                   :506-531
  * boundary terms (:400-470): ``_init_boundary_terms`` (face blocks, 2D
    face mass kron(m1, m1), m1 = B^T W B, and its lump), ``_apply_absorbing``
    (:432-439), the free-surface lumped mass (:268-276), ``bottom_face_load``
    (:441-460), ``surface_height`` (:462-470)
  * ``rk4_step`` with forcing (:506-531)
  * counters: flops of the contractions (tensor.py:204-205), d_reads of
    ``_dfactors`` (:280-286)

Batched over elements with ``bp.chain_batched`` (bit-identical to the
reference's per-element ``_chain``).  On the reference's axis-aligned boxes
``dmat`` is diagonal, so the einsum contractions ``qsr,sq->rq`` /
``qsr,rq->sq`` reduce to one product per entry plus exact zeros, and the
restatement is bit-identical to the reference (pinned by
tests/golden/golden_mixed.npz).
"""

from __future__ import annotations

import numpy as np

from . import bp


class MixedProblem:
    """H1 pressure (order_p) x L2 velocity (order_u) on a structured box."""

    def __init__(self, nx, ny, nz, order_p=4, order_u=3, q=5, extents=(1.0, 1.0, 1.0),
                 rho=1.0, bulk=1.0, coupling_scale=1.0):
        self.n = (nx, ny, nz)
        self.nel = nx * ny * nz
        self.dp, self.du, self.q = order_p + 1, order_u + 1, q
        self.Bp, self.Gp, self.w = bp.basis_tables(self.dp, q)
        self.Bu, self.Gu, _ = bp.basis_tables(self.du, q)
        self.jd, self.detj = bp.jacobian(nx, ny, nz, extents)
        self.jinv = 1.0 / self.jd
        self.wdet = bp.quad_weights_3d(self.w) * self.detj          # operator.py:171-172
        self.dm = np.stack([self.wdet * self.jinv[s] for s in range(3)])  # diagonal of dmat
        self.ids = bp.gather_ids(nx, ny, nz, self.dp)
        self.ndof_p = bp.num_dofs(nx, ny, nz, self.dp)
        self.rho = np.broadcast_to(np.asarray(rho, dtype=np.float64), (self.nel,)).copy()
        self.kinv = 1.0 / np.broadcast_to(np.asarray(bulk, dtype=np.float64), (self.nel,))
        self.cs = float(coupling_scale)
        q3 = q ** 3
        # lumped diagonals, operator.py:179-190
        lu = bp.chain((self.Bu.T,) * 3, self.wdet.copy(), (q, q, q))
        lp = bp.chain((self.Bp.T,) * 3, self.wdet.copy(), (q, q, q))
        self.lump_u = self.rho[:, None] * lu[None, :]
        self.lump_p = bp.scatter_add(self.ids, self.kinv[:, None] * lp[None, :], self.ndof_p)
        assert self.dm.shape == (3, q3)

    @property
    def num_dofs(self) -> int:
        return 3 * self.nel * self.du ** 3 + self.ndof_p

    def tau(self, Pe):
        """_pressure_to_velocity for a batch of gathered pressures (nel, dp^3)
        -> (3, nel, du^3)."""
        dp, du, q = self.dp, self.du, self.q
        A = Pe.reshape(-1, dp, dp, dp)
        out = np.empty((3, Pe.shape[0], du ** 3))
        for r in range(3):
            g = bp.chain_batched([self.Gp if s == r else self.Bp for s in range(3)], A)
            t = self.dm[r].reshape(1, q, q, q) * g
            out[r] = bp.chain_batched((self.Bu.T,) * 3, t).reshape(Pe.shape[0], -1)
        return out

    def vblock(self, U):
        """_velocity_to_pressure for element velocities (3, nel, du^3) ->
        element pressure-test values (nel, dp^3)."""
        du, q = self.du, self.q
        total = None
        for r in range(3):
            uq = bp.chain_batched((self.Bu,) * 3, U[r].reshape(-1, du, du, du))
            t = self.dm[r].reshape(1, q, q, q) * uq
            leg = bp.chain_batched([self.Gp.T if s == r else self.Bp.T for s in range(3)], t)
            total = leg if total is None else total + leg
        return total.reshape(U.shape[1], -1)

    def apply(self, u, p):
        """BlockOperator.apply (operator.py:331-362): (out_u, out_p)."""
        u = np.asarray(u, dtype=np.float64)
        p = np.asarray(p, dtype=np.float64)
        if u.shape != (3, self.nel, self.du ** 3) or p.shape != (self.ndof_p,):
            raise ValueError(f"state dimensions {u.shape}/{p.shape} do not match operator")
        out_u = self.tau(p[self.ids])
        out_p = bp.scatter_add(self.ids, -self.vblock(u), self.ndof_p)
        if self.cs != 1.0:
            out_u *= self.cs
            out_p *= self.cs
        return out_u, out_p

    def fused_normal(self, u):
        """apply_fused_normal (operator.py:364-387): tau(G G^T v(u))."""
        z = bp.scatter_add(self.ids, self.vblock(u), self.ndof_p)
        return self.tau(z[self.ids])

    def mass_inverse(self, ru, rp):
        """apply_mass_inverse (operator.py:391-397)."""
        return ru / self.lump_u[None, :, :], rp / self.lump_p

    def rk4_step(self, u, p, dt, forcing=None, t=0.0):
        """rk4_step (operator.py:506-531); forcing(t) -> (f_u, f_p)."""
        def rhs(time, uu, pp):
            ru, rp = self.apply(uu, pp)
            ru, rp = -ru, -rp
            if forcing is not None:
                fu, fp = forcing(time)
                ru, rp = ru + fu, rp + fp
            return self.mass_inverse(ru, rp)

        k1 = rhs(t, u, p)
        k2 = rhs(t + dt / 2, 1.0 * u + dt / 2 * k1[0], 1.0 * p + dt / 2 * k1[1])
        k3 = rhs(t + dt / 2, 1.0 * u + dt / 2 * k2[0], 1.0 * p + dt / 2 * k2[1])
        k4 = rhs(t + dt, 1.0 * u + dt * k3[0], 1.0 * p + dt * k3[1])
        nu = 1.0 * u + dt / 6 * k1[0] + dt / 3 * k2[0] + dt / 3 * k3[0] + dt / 6 * k4[0]
        np_ = 1.0 * p + dt / 6 * k1[1] + dt / 3 * k2[1] + dt / 3 * k3[1] + dt / 6 * k4[1]
        return nu, np_

    # -- boundary terms (operator.py:400-470) -------------------------------------

    def faces(self, tag):
        """(element, axis, side) of the tagged boundary faces in the
        reference's order (mesh.py:95-119: elements lexicographic, per element
        x-low, x-high, y-low, y-high [absorbing], z-low [bottom], z-high
        [surface])."""
        nx, ny, nz = self.n
        out = []
        for ez in range(nz):
            for ey in range(ny):
                for ex in range(nx):
                    e = ex + nx * (ey + ny * ez)
                    cand = [(ex == 0, 0, 0, "absorbing"), (ex == nx - 1, 0, 1, "absorbing"),
                            (ey == 0, 1, 0, "absorbing"), (ey == ny - 1, 1, 1, "absorbing"),
                            (ez == 0, 2, 0, "bottom"), (ez == nz - 1, 2, 1, "surface")]
                    out += [(e, ax, sd) for hit, ax, sd, tg in cand if hit and tg == tag]
        return out

    def face_local(self, axis, side):
        """_face_local_indices (operator.py:201-210): in-plane order, first
        in-plane index fastest."""
        d = self.dp
        idx = np.arange(d ** 3).reshape((d, d, d), order="F")
        lay = 0 if side == 0 else d - 1
        f = idx[lay, :, :] if axis == 0 else idx[:, lay, :] if axis == 1 else idx[:, :, lay]
        return f.ravel(order="F")

    def area(self, axis):
        h = 2.0 * self.jd
        a, b = [x for x in range(3) if x != axis]
        return (h[a] / 2.0) * (h[b] / 2.0)

    def face_mass2d(self):
        m1 = self.Bp.T @ (self.w[:, None] * self.Bp)
        return np.kron(m1, m1)

    def face_lump2d(self):
        l1 = self.Bp.T @ self.w
        return np.kron(l1, l1)

    def absorbing(self, p, out=None):
        """_apply_absorbing: adds (area/Z) M2d p_face over the lateral faces
        into ``out`` in place (face order, np.add.at, as the reference)."""
        out = np.zeros(self.ndof_p) if out is None else out
        M = self.face_mass2d()
        for e, ax, sd in self.faces("absorbing"):
            z = self.rho[e] * np.sqrt(1.0 / (self.rho[e] * self.kinv[e]))
            g = self.ids[e][self.face_local(ax, sd)]
            np.add.at(out, g, (self.area(ax) / z) * (M @ p[g]))
        return out

    def apply_absorbing(self, u, p):
        """apply with absorbing=True: (v-blocks + absorbing) * coupling_scale."""
        out_u = self.tau(p[self.ids])
        out_p = bp.scatter_add(self.ids, -self.vblock(u), self.ndof_p)
        self.absorbing(p, out_p)
        if self.cs != 1.0:
            out_u *= self.cs
            out_p *= self.cs
        return out_u, out_p

    def surface_lump_p(self, g):
        """lump_p with the free-surface term (operator.py:268-276)."""
        lp = self.lump_p.copy()
        L = self.face_lump2d()
        for e, ax, sd in self.faces("surface"):
            gid = self.ids[e][self.face_local(ax, sd)]
            np.add.at(lp, gid, (1.0 / (self.rho[e] * g)) * (self.area(ax) * L))
        return lp

    def surface_height(self, p, g):
        """surface_height (operator.py:462-470)."""
        vals = [p[self.ids[e][self.face_local(ax, sd)]] / (self.rho[e] * g)
                for e, ax, sd in self.faces("surface")]
        return np.concatenate(vals) if vals else np.zeros(0)

    def bottom_face_load(self, profile):
        """bottom_face_load (operator.py:441-460)."""
        load = np.zeros(self.ndof_p)
        M = self.face_mass2d()
        nodes = bp.gll_points(self.dp)
        h = 2.0 * self.jd
        nx, ny, _ = self.n
        for e, ax, sd in self.faces("bottom"):
            ex, ey = e % nx, (e // nx) % ny
            xs = ex * h[0] + (nodes + 1.0) * 0.5 * h[0]
            ys = ey * h[1] + (nodes + 1.0) * 0.5 * h[1]
            gx, gy = np.meshgrid(xs, ys, indexing="ij")
            vals = np.asarray(profile(gx.ravel(order="F"), gy.ravel(order="F")))
            gid = self.ids[e][self.face_local(ax, sd)]
            np.add.at(load, gid, self.area(ax) * (M @ vals))
        return load

    # -- counters (counters.py, tensor.py:204-205, operator.py:280-286) ------------

    def counts(self, strategy, normal=False):
        """(operator_applies, flops, d_reads) of one apply / apply_fused_normal."""
        def chain(n, m):  # three cyclic contractions n -> m per direction
            return 2 * n * m * (n * n + n * m + m * m)

        flops = 6 * self.nel * (chain(self.dp, self.q) + chain(self.du, self.q))
        per = 9 * self.q ** 3 * self.nel
        d = {"PA": 2 * per, "FusedPA": per}.get(strategy, 0)
        return (0 if normal else 1), flops, d
