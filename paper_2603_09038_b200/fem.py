"""Host-side discretisation setup: box meshes, 1D nodal bases, H1 restriction.

This is the setup half of the drop-in: the objects a ``PAOperator`` is built
from.  They mirror the reference package ``feklab`` so that either set of
objects can be handed to the operator (the operator only duck-types the
attributes used below):

* ``Basis1D`` / ``gll_points`` / ``gauss_points`` restate
  ``feklab/tensor.py:29-122`` with the same NumPy polynomial calls, so the
  tables passed to the CUDA kernels are bit-identical to the reference's
  (checked in ``tests/test_fem_host.py`` against ``tests/golden``).
* ``Mesh`` / ``build_mesh`` restate ``feklab/mesh.py:34-120`` for the
  structured axis-aligned box (vertex/face lists are built lazily; the
  operator only needs ``nx, ny, nz, extents`` and the constant Jacobian).
* ``h1_restriction`` restates ``feklab/mesh.py:144-166`` in closed form
  (vectorised); the device builds the same map in ``fk_restriction_kernel``.

Nothing here runs on the hot path; the apply itself is CUDA only.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class ShapeError(ValueError):
    """Tensor extents and operator dimensions disagree (feklab/tensor.py:20)."""


class GeometryError(ValueError):
    """Degenerate mesh geometry (feklab/mesh.py:16)."""


# ---------------------------------------------------------------------------
# 1D bases  (feklab/tensor.py:29-122)
# ---------------------------------------------------------------------------


def gll_points(n: int, interval: tuple[float, float] = (-1.0, 1.0)) -> np.ndarray:
    """Gauss-Lobatto-Legendre nodes: endpoints and the roots of P'_{n-1}.

    Same construction as feklab/tensor.py:29-41 (monomial form of the
    Legendre derivative, companion-matrix roots), so the nodes agree bitwise.
    """
    if n < 2:
        raise ValueError(f"GLL rule needs at least 2 points, got {n}")
    if n == 2:
        ref = np.array([-1.0, 1.0])
    else:
        leg = np.zeros(n)
        leg[-1] = 1.0
        dpoly = np.polynomial.Polynomial(np.polynomial.legendre.leg2poly(leg)).deriv()
        ref = np.concatenate(([-1.0], np.sort(np.real(dpoly.roots())), [1.0]))
    lo, hi = interval
    return 0.5 * (lo + hi) + 0.5 * (hi - lo) * ref


def gauss_points(n: int, interval: tuple[float, float] = (-1.0, 1.0)):
    """Gauss-Legendre points and weights (feklab/tensor.py:44-48)."""
    x, w = np.polynomial.legendre.leggauss(n)
    lo, hi = interval
    return 0.5 * (lo + hi) + 0.5 * (hi - lo) * x, 0.5 * (hi - lo) * w


def _cardinal_coeffs(nodes: np.ndarray) -> list[np.ndarray]:
    P = np.polynomial.polynomial
    out = []
    for i in range(nodes.size):
        c = P.polyfromroots(np.delete(nodes, i))
        out.append(c / P.polyval(nodes[i], c))
    return out


def lagrange_values(nodes: np.ndarray, points: np.ndarray) -> np.ndarray:
    """L_i(x_a), shape (len(points), len(nodes)) (feklab/tensor.py:62-65)."""
    P = np.polynomial.polynomial
    return np.column_stack([P.polyval(points, c) for c in _cardinal_coeffs(nodes)])


def lagrange_derivatives(nodes: np.ndarray, points: np.ndarray) -> np.ndarray:
    """L_i'(x_a), shape (len(points), len(nodes)) (feklab/tensor.py:68-74)."""
    P = np.polynomial.polynomial
    return np.column_stack(
        [P.polyval(points, P.polyder(c)) for c in _cardinal_coeffs(nodes)]
    )


@dataclass(frozen=True)
class Basis1D:
    """values[a, i] = L_i(x_a) and its derivative table, q rows by d columns."""

    num_dofs_1d: int
    num_quad_1d: int
    values: np.ndarray
    gradients: np.ndarray
    nodes: np.ndarray | None = None
    quad_points: np.ndarray | None = None
    quad_weights: np.ndarray | None = None

    def __post_init__(self):
        q, d = self.num_quad_1d, self.num_dofs_1d
        if self.values.shape != (q, d):
            raise ShapeError(f"values must be {q}x{d}, got {self.values.shape}")
        if self.gradients.shape != (q, d):
            raise ShapeError(f"gradients must be {q}x{d}, got {self.gradients.shape}")

    @classmethod
    def nodal(cls, num_dofs_1d: int, num_quad_1d: int,
              interval: tuple[float, float] = (-1.0, 1.0)) -> "Basis1D":
        nodes = gll_points(num_dofs_1d, interval)
        qpts, qwts = gauss_points(num_quad_1d, interval)
        return cls(num_dofs_1d, num_quad_1d, lagrange_values(nodes, qpts),
                   lagrange_derivatives(nodes, qpts), nodes, qpts, qwts)


# ---------------------------------------------------------------------------
# Structured box mesh  (feklab/mesh.py:34-120)
# ---------------------------------------------------------------------------


@dataclass
class Mesh:
    """Axis-aligned nx*ny*nz box; element e = ex + nx*(ey + ny*ez)."""

    nx: int
    ny: int
    nz: int
    extents: tuple[float, float, float] = (1.0, 1.0, 1.0)
    _vertices: np.ndarray | None = field(default=None, repr=False)

    @property
    def num_elements(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def element_size(self) -> tuple[float, float, float]:
        return (self.extents[0] / self.nx, self.extents[1] / self.ny,
                self.extents[2] / self.nz)

    @property
    def jacobian_diag(self) -> np.ndarray:
        h = self.element_size
        return np.array([h[0] / 2.0, h[1] / 2.0, h[2] / 2.0])

    @property
    def jacobian_det(self) -> float:
        return float(np.prod(self.jacobian_diag))

    def element_coords(self, e: int) -> tuple[int, int, int]:
        return e % self.nx, (e // self.nx) % self.ny, e // (self.nx * self.ny)

    @property
    def vertices(self) -> np.ndarray:
        if self._vertices is None:
            h = self.element_size
            axes = [np.arange(n + 1) * hh for n, hh in zip((self.nx, self.ny, self.nz), h)]
            g = np.meshgrid(*axes, indexing="ij")
            self._vertices = np.column_stack([a.ravel(order="F") for a in g])
        return self._vertices


def build_mesh(nx: int, ny: int, nz: int, extents=(1.0, 1.0, 1.0)) -> Mesh:
    if min(nx, ny, nz) < 1:
        raise GeometryError(f"element counts must be >= 1, got {(nx, ny, nz)}")
    if min(extents) <= 0:
        raise GeometryError(f"domain extents must be positive, got {extents}")
    return Mesh(int(nx), int(ny), int(nz), tuple(float(x) for x in extents))


# ---------------------------------------------------------------------------
# H1 restriction  (feklab/mesh.py:123-166)
# ---------------------------------------------------------------------------


@dataclass
class Restriction:
    num_global: int
    gather_ids: np.ndarray  # (num_elements, d^3) int64

    def gather(self, global_vec: np.ndarray) -> np.ndarray:
        return global_vec[self.gather_ids]

    def scatter_add(self, element_vals: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.zeros(self.num_global)
        np.add.at(out, self.gather_ids.ravel(), element_vals.ravel())
        return out

    def multiplicity(self) -> np.ndarray:
        return self.scatter_add(np.ones(self.gather_ids.shape))


def global_node_counts(nx: int, ny: int, nz: int, d: int) -> tuple[int, int, int]:
    return nx * (d - 1) + 1, ny * (d - 1) + 1, nz * (d - 1) + 1


def h1_gather_ids(nx: int, ny: int, nz: int, d: int, ez_range: tuple[int, int] | None = None) -> np.ndarray:
    """Closed form of feklab/mesh.py:157-164: local node i + d*(j + d*k) of
    element (ex, ey, ez) maps to gi + npx*(gj + npy*gk), gi = ex*(d-1)+i ...

    ez_range selects a contiguous z-slab of element layers [z0, z1) (rows
    z0*nx*ny .. z1*nx*ny of the full map, since elements are z-slowest).
    """
    npx, npy, _ = global_node_counts(nx, ny, nz, d)
    z0, z1 = (0, nz) if ez_range is None else ez_range
    ex = np.arange(nx, dtype=np.int64)
    ey = np.arange(ny, dtype=np.int64)
    ez = np.arange(z0, z1, dtype=np.int64)
    l = np.arange(d, dtype=np.int64)
    # element-major (ez, ey, ex), then local (k, j, i) with i fastest
    gi = (ex[None, None, :, None, None, None] * (d - 1) + l[None, None, None, None, None, :])
    gj = (ey[None, :, None, None, None, None] * (d - 1) + l[None, None, None, None, :, None])
    gk = (ez[:, None, None, None, None, None] * (d - 1) + l[None, None, None, :, None, None])
    ids = gi + npx * (gj + npy * gk)
    return ids.reshape((z1 - z0) * ny * nx, d ** 3)


def h1_restriction(mesh, num_dofs_1d: int) -> Restriction:
    d = num_dofs_1d
    npx, npy, npz = global_node_counts(mesh.nx, mesh.ny, mesh.nz, d)
    return Restriction(npx * npy * npz, h1_gather_ids(mesh.nx, mesh.ny, mesh.nz, d))


def h1_node_coords(mesh, nodes_1d: np.ndarray) -> np.ndarray:
    """Physical coordinates of the global nodes, x fastest (feklab/mesh.py:169-188)."""
    d = nodes_1d.size
    axes = []
    for n_el, hh in zip((mesh.nx, mesh.ny, mesh.nz), mesh.element_size):
        pts = np.empty(n_el * (d - 1) + 1)
        for e in range(n_el):
            pts[e * (d - 1): e * (d - 1) + d] = e * hh + (nodes_1d + 1.0) * 0.5 * hh
        axes.append(pts)
    g = np.meshgrid(*axes, indexing="ij")
    return np.column_stack([a.ravel(order="F") for a in g])


def boundary_dofs(nx: int, ny: int, nz: int, d: int) -> np.ndarray:
    """Global ids of every node on the six faces of the box (sorted, int64)."""
    npx, npy, npz = global_node_counts(nx, ny, nz, d)
    gi = np.arange(npx)
    gj = np.arange(npy)
    gk = np.arange(npz)
    on = ((gi[None, None, :] == 0) | (gi[None, None, :] == npx - 1)
          | (gj[None, :, None] == 0) | (gj[None, :, None] == npy - 1)
          | (gk[:, None, None] == 0) | (gk[:, None, None] == npz - 1))
    return np.flatnonzero(on.ravel()).astype(np.int64)


# ---------------------------------------------------------------------------
# Instrumentation  (feklab/counters.py:8-29)
# ---------------------------------------------------------------------------


@dataclass
class Counters:
    flops: int = 0
    d_reads: int = 0
    operator_applies: int = 0
    extra: dict = field(default_factory=dict)

    def reset(self) -> None:
        self.flops = 0
        self.d_reads = 0
        self.operator_applies = 0
        self.extra.clear()

    def bump(self, key: str, amount: int = 1) -> None:
        self.extra[key] = self.extra.get(key, 0) + amount
