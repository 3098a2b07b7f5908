"""NumPy restatement of the reference's BP1/BP3 path — TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py for scope and pinning.  Every function cites the
reference (``/root/reference/pkg/src/feklab``) file:line it restates.

Tensor convention (feklab/tensor.py:132-139): an element tensor is a flat
FP64 vector whose first extent is fastest.  Batched element tensors are
C-order arrays ``A[e, i2, i1, i0]`` (same memory order per element).
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# Bases (feklab/tensor.py:29-122)
# ---------------------------------------------------------------------------


def gll_points(n: int) -> np.ndarray:
    """feklab/tensor.py:29-41 on [-1, 1]."""
    if n == 2:
        pts = np.array([-1.0, 1.0])
    else:
        inner = np.polynomial.Polynomial(
            np.polynomial.legendre.leg2poly([0.0] * (n - 1) + [1.0])).deriv().roots()
        pts = np.concatenate(([-1.0], np.sort(np.real(inner)), [1.0]))
    return 0.0 + 1.0 * pts


def basis_tables(d: int, q: int):
    """(B, G, w): values/gradients (q x d) and Gauss weights, as
    Basis1D.nodal (feklab/tensor.py:101-119) builds them."""
    P = np.polynomial.polynomial
    nodes = gll_points(d)
    x, w = np.polynomial.legendre.leggauss(q)
    qpts, qw = 0.0 + 1.0 * x, 1.0 * w
    coeffs = []
    for i, xi in enumerate(nodes):
        c = P.polyfromroots(np.delete(nodes, i))
        coeffs.append(c / P.polyval(xi, c))
    B = np.column_stack([P.polyval(qpts, c) for c in coeffs])
    G = np.column_stack([P.polyval(qpts, P.polyder(c)) for c in coeffs])
    return B, G, qw


def node_coords_1d(d: int) -> np.ndarray:
    return gll_points(d)


# ---------------------------------------------------------------------------
# Mesh data (feklab/mesh.py:44-64, 144-166; operator.py:132-134)
# ---------------------------------------------------------------------------


def jacobian(nx, ny, nz, extents=(1.0, 1.0, 1.0)):
    """(jacobian_diag, jacobian_det) as feklab/mesh.py:56-64."""
    h = (extents[0] / nx, extents[1] / ny, extents[2] / nz)
    jd = np.array([h[0] / 2.0, h[1] / 2.0, h[2] / 2.0])
    return jd, float(np.prod(jd))


def gather_ids(nx, ny, nz, d, ez_range=None) -> np.ndarray:
    """feklab/mesh.py:157-164: gather[e, i + d(j + d k)] =
    (ex(d-1)+i) + npx((ey(d-1)+j) + npy(ez(d-1)+k)), e = ex + nx(ey + ny ez)."""
    npx, npy = nx * (d - 1) + 1, ny * (d - 1) + 1
    z0, z1 = (0, nz) if ez_range is None else ez_range
    ez, ey, ex = np.meshgrid(np.arange(z0, z1), np.arange(ny), np.arange(nx), indexing="ij")
    k, j, i = np.meshgrid(np.arange(d), np.arange(d), np.arange(d), indexing="ij")
    gi = ex.reshape(-1, 1) * (d - 1) + i.reshape(1, -1)
    gj = ey.reshape(-1, 1) * (d - 1) + j.reshape(1, -1)
    gk = ez.reshape(-1, 1) * (d - 1) + k.reshape(1, -1)
    return (gi + npx * (gj + npy * gk)).astype(np.int64)


def gather_ids_elements(nx, ny, nz, d, e0, e1) -> np.ndarray:
    """Rows e0..e1-1 of gather_ids (same closed form, any element range)."""
    npx, npy = nx * (d - 1) + 1, ny * (d - 1) + 1
    e = np.arange(e0, e1, dtype=np.int64)
    ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
    k, j, i = np.meshgrid(np.arange(d), np.arange(d), np.arange(d), indexing="ij")
    gi = ex[:, None] * (d - 1) + i.reshape(1, -1)
    gj = ey[:, None] * (d - 1) + j.reshape(1, -1)
    gk = ez[:, None] * (d - 1) + k.reshape(1, -1)
    return gi + npx * (gj + npy * gk)


def num_dofs(nx, ny, nz, d) -> int:
    return (nx * (d - 1) + 1) * (ny * (d - 1) + 1) * (nz * (d - 1) + 1)


def quad_weights_3d(w: np.ndarray) -> np.ndarray:
    """feklab/operator.py:132-134."""
    return np.kron(w, np.kron(w, w))


def scatter_add(ids: np.ndarray, vals: np.ndarray, n: int) -> np.ndarray:
    """feklab/mesh.py:133-137 (np.add.at, element-major order)."""
    out = np.zeros(n)
    np.add.at(out, ids.ravel(), vals.ravel())
    return out


# ---------------------------------------------------------------------------
# Cyclic contractions (feklab/tensor.py:177-283)
# ---------------------------------------------------------------------------


def contract_cyclic(m: np.ndarray, data: np.ndarray, extents):
    """Single element, feklab/tensor.py:177-210: out(j,k,a) = sum_i m[a,i] x(i,j,k),
    accumulated over ascending i with separate multiply and add."""
    q, d = m.shape
    e0, e1, e2 = extents
    assert e0 == d
    x2 = data.reshape(d, e1 * e2, order="F")
    out2 = np.zeros((e1 * e2, q))
    for i in range(d):
        out2 += np.multiply.outer(x2[i], m[:, i])
    return out2.ravel(order="F"), (e1, e2, q)


def chain(mats, data, extents):
    for m in mats:
        data, extents = contract_cyclic(m, data, extents)
    return data


def contract_cyclic_batched(m: np.ndarray, A: np.ndarray) -> np.ndarray:
    """Batched restatement: A[e, i2, i1, i0] -> out[e, a, i2, i1]; per output
    entry the same ascending-i multiply-then-add sequence as contract_cyclic,
    hence bit-identical."""
    q, d = m.shape
    assert A.shape[3] == d
    out = np.zeros((A.shape[0], q, A.shape[1], A.shape[2]))
    for i in range(d):
        out += A[:, None, :, :, i] * m[None, :, i, None, None]
    return out


def chain_batched(mats, A):
    for m in mats:
        A = contract_cyclic_batched(m, A)
    return A


# ---------------------------------------------------------------------------
# BP1 / BP3 element operators (SURVEY.md §8c recipe)
# ---------------------------------------------------------------------------


def bp1_element(B, wdet, xe):
    """apply_basis_transpose_3d(wdet * apply_basis_3d(x)) (tensor.py:220-241)."""
    d, q = B.shape[1], B.shape[0]
    u = chain((B, B, B), xe, (d, d, d))
    return chain((B.T, B.T, B.T), wdet * u, (q, q, q))


def bp3_element(B, G, wdet, jinv, xe):
    """Gradient legs (tensor.py:244-260), t_s = wdet*jinv_s^2*g_s,
    transpose legs summed in order r = 0, 1, 2 (tensor.py:263-283)."""
    d, q = B.shape[1], B.shape[0]
    g = [chain([G if s == r else B for s in range(3)], xe, (d, d, d)) for r in range(3)]
    t = [wdet * jinv[s] ** 2 * g[s] for s in range(3)]
    total = None
    for r in range(3):
        leg = chain([G.T if s == r else B.T for s in range(3)], t[r], (q, q, q))
        if total is None:
            total = leg
        else:
            total += leg
    return total


def bp1_batched(B, wdet, Xe):
    d, q = B.shape[1], B.shape[0]
    A = Xe.reshape(-1, d, d, d)
    u = chain_batched((B, B, B), A)
    u = wdet.reshape(1, q, q, q) * u
    return chain_batched((B.T, B.T, B.T), u).reshape(Xe.shape[0], -1)


def bp3_batched(B, G, wdet, jinv, Xe):
    d, q = B.shape[1], B.shape[0]
    A = Xe.reshape(-1, d, d, d)
    total = None
    for r in range(3):
        g = chain_batched([G if s == r else B for s in range(3)], A)
        t = (wdet * jinv[r] ** 2).reshape(1, q, q, q) * g
        leg = chain_batched([G.T if s == r else B.T for s in range(3)], t)
        total = leg if total is None else total + leg
    return total.reshape(Xe.shape[0], -1)


class Problem:
    """Everything the oracle needs for one (mesh, p, q, kind) configuration."""

    def __init__(self, kind, nx, ny, nz, p, q=None, extents=(1.0, 1.0, 1.0), ez_range=None):
        assert kind in ("mass", "diffusion")
        self.kind = kind
        self.nx, self.ny, self.nz = nx, ny, nz
        self.p = p
        self.d = p + 1
        self.q = q if q is not None else p + 2
        self.B, self.G, self.w = basis_tables(self.d, self.q)
        self.jd, self.detj = jacobian(nx, ny, nz, extents)
        self.jinv = 1.0 / self.jd
        self.wdet = quad_weights_3d(self.w) * self.detj
        self.ez_range = ez_range
        self.ids = gather_ids(nx, ny, nz, self.d, ez_range)
        self.ndof = num_dofs(nx, ny, nz, self.d)

    # -- operator ---------------------------------------------------------

    def element_apply(self, Xe, batched=True):
        if batched:
            if self.kind == "mass":
                return bp1_batched(self.B, self.wdet, Xe)
            return bp3_batched(self.B, self.G, self.wdet, self.jinv, Xe)
        out = np.empty((Xe.shape[0], self.d ** 3))
        for e in range(Xe.shape[0]):
            if self.kind == "mass":
                out[e] = bp1_element(self.B, self.wdet, Xe[e].copy())
            else:
                out[e] = bp3_element(self.B, self.G, self.wdet, self.jinv, Xe[e].copy())
        return out

    def apply(self, x, batched=True, chunk=4096):
        """y = G^T (B^T D B) G x; element values are produced in chunks and
        scattered once in element-major order, as Restriction.scatter_add."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.ndof,):
            raise ValueError(f"vector dimensions {x.shape} do not match operator ({self.ndof},)")
        ye = np.empty(self.ids.shape)
        for s in range(0, self.ids.shape[0], chunk):
            ye[s:s + chunk] = self.element_apply(x[self.ids[s:s + chunk]], batched)
        return scatter_add(self.ids, ye, self.ndof)

    def diagonal(self):
        """Assembled diag(A): transpose chains with squared tables applied to
        the (diagonal) PA data, then scatter_add."""
        B2, G2 = self.B * self.B, self.G * self.G
        q = self.q
        if self.kind == "mass":
            de = chain((B2.T, B2.T, B2.T), self.wdet.copy(), (q, q, q))
        else:
            de = None
            for r in range(3):
                t = self.wdet * self.jinv[r] ** 2
                leg = chain([G2.T if s == r else B2.T for s in range(3)], t, (q, q, q))
                de = leg if de is None else de + leg
        nel = self.ids.shape[0]
        return scatter_add(self.ids, np.broadcast_to(de, (nel, de.size)), self.ndof)

    def boundary(self):
        npx, npy, npz = (self.nx * self.p + 1, self.ny * self.p + 1, self.nz * self.p + 1)
        gk, gj, gi = np.meshgrid(np.arange(npz), np.arange(npy), np.arange(npx), indexing="ij")
        on = (gi == 0) | (gi == npx - 1) | (gj == 0) | (gj == npy - 1) | (gk == 0) | (gk == npz - 1)
        return np.flatnonzero(on.ravel())

    def constrained_apply(self, x, ess):
        """MFEM ConstrainedOperator (DIAG_ONE): zero essential inputs, apply,
        copy essential inputs to the output."""
        xz = np.array(x, dtype=np.float64)
        xz[ess] = 0.0
        y = self.apply(xz)
        y[ess] = x[ess]
        return y

    def pcg(self, b, iters=100, ess=None, rtol=0.0):
        """Jacobi-preconditioned CG, MFEM CGSolver semantics, x0 = 0.
        Returns (x, history) with history[k] = sqrt(r_k . z_k)."""
        if ess is None:
            ess = self.boundary()
        dinv = 1.0 / self.diagonal()
        dinv[ess] = 1.0
        A = lambda v: self.constrained_apply(v, ess)
        x = np.zeros(self.ndof)
        r = np.array(b, dtype=np.float64)
        z = dinv * r
        p = z.copy()
        nom = float(r @ z)
        hist = [np.sqrt(nom)]
        # MFEM CGSolver: converged when nom <= max(rtol^2 nom0, abs_tol^2)
        # (abs_tol = 0), which includes an exactly zero residual; break on
        # p.Ap == 0
        stop = rtol * rtol * nom
        if nom <= stop:
            return x, np.array(hist)
        for _ in range(iters):
            Ap = A(p)
            den = float(p @ Ap)
            if den == 0.0:
                break
            alpha = nom / den
            x += alpha * p
            r -= alpha * Ap
            z = dinv * r
            betanom = float(r @ z)
            hist.append(np.sqrt(betanom))
            if betanom <= stop:
                break
            beta = betanom / nom
            p = z + beta * p
            nom = betanom
        return x, np.array(hist)
