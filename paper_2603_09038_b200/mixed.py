"""Acoustic-gravity block operator on B200.

Drop-in sibling of ``feklab.operator.BlockOperator`` (operator.py:221-397)
for the FusedPA / PA strategies: the coupled first-order wave operator with a
continuous H1 pressure (``order_p``) and discontinuous L2 velocity
(``order_u``), evaluated by one fused sm_100a kernel per apply that reads the
quadrature factors ``dmat`` once for both off-diagonal blocks
(libfk_b200.so, ``fk_mix_*`` in include/fk.h).  ``rk4_step`` mirrors
operator.py:506-531 and ``MixedOperator.rk4`` runs whole steps on the device.

States are ``State(u, p)`` with ``u`` of shape (3, nel, (order_u+1)^3) and
``p`` of length ``num_p`` — NumPy arrays (host; copied in and out) or CUDA
float64 tensors (stay on the device); the reference's own ``State`` objects
are accepted (duck-typed ``.u`` / ``.p``).  No CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fem import Basis1D, Counters, h1_gather_ids

# PA / FusedPA: stored dmat (one fused pass reads it once for both blocks);
# MF / FusedMF: dmat recomputed in the kernel (operator.py:16-19, 280-286)
STRATEGIES = ("PA", "FusedPA", "MF", "FusedMF")


def _torch():
    import torch

    return torch


class DivergenceError(FloatingPointError):
    """Time stepping produced non-finite values (operator.py:52-53)."""


@dataclass
class State:
    """Velocity blocks (3, elements, local dofs) plus pressure dofs (operator.py:63-90)."""

    u: object
    p: object

    def copy(self) -> "State":
        return State(self.u.copy() if isinstance(self.u, np.ndarray) else self.u.clone(),
                     self.p.copy() if isinstance(self.p, np.ndarray) else self.p.clone())

    @property
    def num_dofs(self) -> int:
        return int(np.prod(self.u.shape)) + int(self.p.shape[0])


class MixedOperator:
    """``BlockOperator(mesh, order_p, order_u, num_quad_1d, strategy, ...)`` on B200.

    Supported: order_u = order_p - 1, num_quad_1d = order_p + 1, order_p = 2..8
    (the reference default 4/3/5), scalar or per-element rho / bulk modulus,
    coupling_scale, absorbing lateral faces (applied on the device inside
    every apply and RK4 stage, :357-358, 432-439), free-surface gravity
    (lumped-mass term, :268-276; ``surface_height``), ``bottom_face_load``
    (:441-460) and forced RK4 (:506-531).  strategy MF / FusedMF recomputes
    dmat in the kernel.  Counters follow the reference: one operator_apply
    and the contraction flops per apply, d_reads 2x / 1x / 0 of the stored
    dmat for PA / FusedPA / MF (``_dfactors``, :280-286).
    """

    def __init__(self, mesh, order_p: int = 4, order_u: int = 3, num_quad_1d: int = 5,
                 strategy: str = "FusedPA", rho=1.0, bulk_modulus=1.0,
                 coupling_scale: float = 1.0, absorbing: bool = False,
                 surface_gravity=None, counters: Counters | None = None, device=None,
                 stream=None):
        if strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
        if surface_gravity is not None and not float(surface_gravity) > 0:
            raise ValueError("surface gravity must be positive")
        self.absorbing = bool(absorbing)
        self.surface_gravity = None if surface_gravity is None else float(surface_gravity)
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("MixedOperator needs a CUDA device (there is no CPU fallback)")
        lib = _lib.load()
        self._lib = lib
        self.mesh = mesh
        self.strategy = strategy
        self.coupling_scale = float(coupling_scale)
        self.counters = counters if counters is not None else Counters()
        self.basis_p = Basis1D.nodal(order_p + 1, num_quad_1d)
        self.basis_u = Basis1D.nodal(order_u + 1, num_quad_1d)
        self.order_p, self.order_u, self.num_quad_1d = int(order_p), int(order_u), int(num_quad_1d)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        with torch.cuda.device(self.device):
            self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        nel = mesh.nx * mesh.ny * mesh.nz
        self._tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in
                      (self.basis_p.values, self.basis_p.gradients, self.basis_u.values,
                       self.basis_p.quad_weights)]
        rho_a = np.broadcast_to(np.asarray(rho, dtype=np.float64), (nel,)).copy()
        bulk_a = np.broadcast_to(np.asarray(bulk_modulus, dtype=np.float64), (nel,)).copy()
        if np.any(rho_a <= 0) or np.any(bulk_a <= 0):
            raise ValueError("density and bulk modulus must be positive")
        self._rho, self._bulk = rho_a, bulk_a
        desc = _lib.FkMixDesc()
        desc.order_p, desc.order_u, desc.num_quad_1d = self.order_p, self.order_u, self.num_quad_1d
        desc.nx, desc.ny, desc.nz = mesh.nx, mesh.ny, mesh.nz
        jd = np.asarray(mesh.jacobian_diag, dtype=np.float64)
        for s in range(3):
            desc.jac_diag[s] = float(jd[s])
        desc.jac_det = float(mesh.jacobian_det)
        pd = ctypes.POINTER(ctypes.c_double)
        desc.Bp, desc.Gp, desc.Bu, desc.w = (t.ctypes.data_as(pd) for t in self._tabs)
        desc.rho = rho_a.ctypes.data_as(pd)
        desc.bulk = bulk_a.ctypes.data_as(pd)
        desc.rho_scalar = desc.bulk_scalar = 1.0
        desc.coupling_scale = self.coupling_scale
        desc.matrix_free = 1 if strategy in ("MF", "FusedMF") else 0
        desc.absorbing = 1 if self.absorbing else 0
        desc.surface_gravity = 0.0 if self.surface_gravity is None else self.surface_gravity
        desc.device = self.device.index
        desc.stream = ctypes.c_void_p(self._stream.cuda_stream)
        h = ctypes.c_void_p()
        _lib.check(lib.fk_mix_create(ctypes.byref(h), ctypes.byref(desc)))
        self._h = h
        _lib.check(lib.fk_mix_setup(self._h))
        info = _lib.FkMixInfo()
        _lib.check(lib.fk_mix_get_info(self._h, ctypes.byref(info)))
        self.info = info
        self.num_elements = int(info.nel)
        self.num_p = int(info.ndof_p)
        self.num_dofs_u_local = (self.order_u + 1) ** 3
        self.num_dofs = int(info.ndof_u) + self.num_p
        self._zero_u = None
        # reference counter semantics (counters.py; tensor.py:204-205 counts
        # 2 d q e1 e2 per contraction; _dfactors :280-286 counts dmat reads)
        chain = lambda n, m: 2 * n * m * (n * n + n * m + m * m)  # noqa: E731
        dp, du, q = self.order_p + 1, self.order_u + 1, self.num_quad_1d
        self.flops_per_apply = 6 * self.num_elements * (chain(dp, q) + chain(du, q))
        per = 9 * q ** 3 * self.num_elements
        self.d_reads_per_apply = {"PA": 2 * per, "FusedPA": per}.get(strategy, 0)

    # -- lifecycle ------------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.fk_mix_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch(self) -> tuple[int, int, int]:
        return self.info.elems_per_block, self.info.threads_per_block, self.info.blocks

    # -- states ---------------------------------------------------------------

    @property
    def u_shape(self) -> tuple[int, int, int]:
        return (3, self.num_elements, self.num_dofs_u_local)

    def zero_state(self, device: bool = False) -> State:
        if device:
            torch = _torch()
            z = lambda *s: torch.zeros(*s, dtype=torch.float64, device=self.device)  # noqa: E731
            return State(z(*self.u_shape), z(self.num_p))
        return State(np.zeros(self.u_shape), np.zeros(self.num_p))

    def _check(self, state) -> None:
        u, p = state.u, state.p
        if tuple(u.shape) != self.u_shape or tuple(p.shape) != (self.num_p,):
            raise ValueError(f"state dimensions {tuple(u.shape)}/{tuple(p.shape)} do not match "
                             f"operator {self.u_shape}/{(self.num_p,)}")

    def _dev(self, a):
        torch = _torch()
        if isinstance(a, np.ndarray):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)
        if a.dtype != torch.float64 or a.device != self.device or not a.is_contiguous():
            raise ValueError("device arrays must be contiguous float64 on the operator's device")
        return a

    # -- operator application ---------------------------------------------------

    def apply(self, state, out: State | None = None) -> State:
        """Residual of the coupling operator acting on [u, p] (operator.py:331-362)."""
        self._check(state)
        torch = _torch()
        host_out = out is not None and isinstance(out.u, np.ndarray)
        if out is not None:
            self._check(out)
            for name, a in (("out.u", out.u), ("out.p", out.p)):
                if isinstance(a, np.ndarray):
                    if a.dtype != np.float64 or not a.flags.c_contiguous or not a.flags.writeable:
                        raise ValueError(f"{name} must be a writeable C-contiguous float64 array")
                elif a.dtype != torch.float64 or a.device != self.device or not a.is_contiguous():
                    raise ValueError(f"{name} must be a contiguous float64 tensor on {self.device}")
        self._count(1)
        host = isinstance(state.u, np.ndarray)
        u, p = self._dev(state.u), self._dev(state.p)
        dev_out = out is not None and not host_out
        ou = self._dev(out.u) if dev_out else torch.empty_like(u)
        op = self._dev(out.p) if dev_out else torch.empty_like(p)
        _lib.check(self._lib.fk_mix_apply(self._h, u.data_ptr(), p.data_ptr(), ou.data_ptr(),
                                          op.data_ptr()))
        if host_out:  # NumPy out buffers are filled in place
            out.u[...] = ou.cpu().numpy()
            out.p[...] = op.cpu().numpy()
            return out
        if dev_out:
            return out
        if host:
            return State(ou.cpu().numpy(), op.cpu().numpy())
        return State(ou, op)

    __call__ = apply

    def _count(self, applies: int, normal: int = 0) -> None:
        """applies: BlockOperator.apply calls; normal: apply_fused_normal calls
        (which the reference does not count as operator applies)."""
        self.counters.operator_applies += applies
        self.counters.flops += (applies + normal) * self.flops_per_apply
        self.counters.d_reads += (applies + normal) * self.d_reads_per_apply

    def apply_fused_normal(self, x_u):
        """Velocity -> assembled pressure -> velocity (operator.py:364-387)."""
        host = isinstance(x_u, np.ndarray)
        if tuple(x_u.shape) != self.u_shape:
            raise ValueError(f"velocity dimensions {tuple(x_u.shape)} do not match {self.u_shape}")
        u = self._dev(x_u)
        out = _torch().empty_like(u)
        self._count(0, 1)
        _lib.check(self._lib.fk_mix_fused_normal(self._h, u.data_ptr(), out.data_ptr()))
        return out.cpu().numpy() if host else out

    def apply_mass_inverse(self, residual) -> State:
        """u / lump_u, p / lump_p (operator.py:391-397)."""
        self._check(residual)
        host = isinstance(residual.u, np.ndarray)
        ru, rp = self._dev(residual.u), self._dev(residual.p)
        u, p = _torch().empty_like(ru), _torch().empty_like(rp)
        _lib.check(self._lib.fk_mix_mass_inverse(self._h, ru.data_ptr(), rp.data_ptr(),
                                                 u.data_ptr(), p.data_ptr()))
        return State(u.cpu().numpy(), p.cpu().numpy()) if host else State(u, p)

    def lumped(self):
        """(lump_u (nel, du^3), lump_p (num_p)) as NumPy arrays (QuadData.lump_u / lump_p)."""
        torch = _torch()
        lu = torch.empty((self.num_elements, self.num_dofs_u_local), dtype=torch.float64,
                         device=self.device)
        lp = torch.empty(self.num_p, dtype=torch.float64, device=self.device)
        _lib.check(self._lib.fk_mix_lumped(self._h, lu.data_ptr(), lp.data_ptr()))
        return lu.cpu().numpy(), lp.cpu().numpy()

    def restriction_ids(self) -> np.ndarray:
        d3 = (self.order_p + 1) ** 3
        out = np.empty((self.num_elements, d3), dtype=np.int64)
        _lib.check(self._lib.fk_mix_restriction(self._h, out.ctypes.data_as(
            ctypes.POINTER(ctypes.c_int64))))
        return out

    def rk4(self, state, dt: float, steps: int = 1) -> State:
        """``steps`` RK4 steps (rk4_step, operator.py:506-531, no forcing) on the
        device, four fused applies per step; returns the new state."""
        self._check(state)
        if not dt > 0:
            raise ValueError(f"dt must be positive, got {dt}")
        host = isinstance(state.u, np.ndarray)
        u, p = self._dev(state.u).clone(), self._dev(state.p).clone()
        self._count(4 * int(steps))
        _lib.check(self._lib.fk_mix_rk4(self._h, u.data_ptr(), p.data_ptr(), float(dt), int(steps)))
        torch = _torch()
        if not (bool(torch.isfinite(u).all()) and bool(torch.isfinite(p).all())):
            raise DivergenceError(f"non-finite state after {steps} step(s)")
        return State(u.cpu().numpy(), p.cpu().numpy()) if host else State(u, p)

    def time_apply(self, state: State, out: State, reps: int) -> tuple[float, float]:
        fa, fk = ctypes.c_double(), ctypes.c_double()
        _lib.check(self._lib.fk_mix_time_apply(self._h, state.u.data_ptr(), state.p.data_ptr(),
                                               out.u.data_ptr(), out.p.data_ptr(), int(reps),
                                               ctypes.byref(fa), ctypes.byref(fk)))
        return fa.value, fk.value

    # -- algorithmic work (bench roofline) ---------------------------------------

    @property
    def bytes_per_apply(self) -> int:
        """u read + out_u write (48 du^3 per element), p read + out_p write
        (16 per H1 dof), dmat (72 q^3; not for MF), int32 map (4 dp^3) per element."""
        du3, dp3, q3 = (self.order_u + 1) ** 3, (self.order_p + 1) ** 3, self.num_quad_1d ** 3
        dm = 0 if self.strategy in ("MF", "FusedMF") else 72 * q3
        return self.num_elements * (48 * du3 + dm + 4 * dp3) + 16 * self.num_p

    def gather_ids(self) -> np.ndarray:
        return h1_gather_ids(self.mesh.nx, self.mesh.ny, self.mesh.nz, self.order_p + 1)

    # -- boundary terms (operator.py:400-470) ------------------------------------

    def _face_ids(self, ez: int, side: int) -> np.ndarray:
        """(nx*ny, dp^2) global pressure ids of the z-faces of element layer
        ``ez`` (side 0 low, 1 high), faces x-fastest, face nodes first
        in-plane index fastest (_face_local_indices, :201-210)."""
        d, nx, ny = self.order_p + 1, self.mesh.nx, self.mesh.ny
        npx, npy = nx * (d - 1) + 1, ny * (d - 1) + 1
        ey, ex = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        b, a = np.meshgrid(np.arange(d), np.arange(d), indexing="ij")
        gi = ex.reshape(-1, 1) * (d - 1) + a.reshape(1, -1)
        gj = ey.reshape(-1, 1) * (d - 1) + b.reshape(1, -1)
        gk = ez * (d - 1) + (d - 1 if side else 0)
        return gi + npx * (gj + npy * gk)

    def bottom_face_load(self, profile) -> np.ndarray:
        """Assembled load of a normal-velocity profile(x, y) on the bottom
        face (operator.py:441-460): the profile is evaluated per bottom face
        at its node positions (host callable), the face mass pairing and the
        assembly run on the device.  Returns a NumPy vector of num_p."""
        torch = _torch()
        d, nx, ny = self.order_p + 1, self.mesh.nx, self.mesh.ny
        nodes = np.asarray(self.basis_p.nodes, dtype=np.float64)
        h = 2.0 * np.asarray(self.mesh.jacobian_diag, dtype=np.float64)
        vals = np.empty((nx * ny, d * d))
        for f in range(nx * ny):
            ex, ey = f % nx, f // nx
            xs = ex * h[0] + (nodes + 1.0) * 0.5 * h[0]
            ys = ey * h[1] + (nodes + 1.0) * 0.5 * h[1]
            gx, gy = np.meshgrid(xs, ys, indexing="ij")
            vals[f] = np.asarray(profile(gx.ravel(order="F"), gy.ravel(order="F")), dtype=np.float64)
        v = torch.as_tensor(vals, device=self.device)
        load = torch.empty(self.num_p, dtype=torch.float64, device=self.device)
        _lib.check(self._lib.fk_mix_bottom_load(self._h, v.data_ptr(), load.data_ptr()))
        return load.cpu().numpy()

    def surface_height(self, state) -> np.ndarray:
        """Free-surface elevation p / (rho g) at the surface-face nodes
        (operator.py:462-470), faces x-fastest."""
        if self.surface_gravity is None:
            raise ValueError("operator was built without surface gravity")
        torch = _torch()
        ids = self._face_ids(self.mesh.nz - 1, 1)
        top = np.arange(self.mesh.nx * self.mesh.ny) + self.mesh.nx * self.mesh.ny * (self.mesh.nz - 1)
        p = self._dev(state.p)
        vals = p[torch.as_tensor(ids.ravel(), device=self.device)].reshape(ids.shape)
        rho = torch.as_tensor(self._rho[top], device=self.device)
        return (vals / (rho[:, None] * self.surface_gravity)).reshape(-1).cpu().numpy()

    def rk4_forced(self, state, dt: float, f0, fh, f1) -> State:
        """One RK4 step with forcing values at t, t + dt/2, t + dt (States)."""
        self._check(state)
        torch = _torch()
        host = isinstance(state.u, np.ndarray)
        u, p = self._dev(state.u).clone(), self._dev(state.p).clone()
        packed = []
        for f in (f0, fh, f1):
            packed.append(torch.cat([self._dev(f.u).reshape(-1), self._dev(f.p).reshape(-1)]))
        self._count(4)
        _lib.check(self._lib.fk_mix_rk4_forced(self._h, u.data_ptr(), p.data_ptr(), float(dt),
                                               *(t.data_ptr() for t in packed)))
        if not (bool(torch.isfinite(u).all()) and bool(torch.isfinite(p).all())):
            raise DivergenceError("non-finite state after the forced step")
        return State(u.cpu().numpy(), p.cpu().numpy()) if host else State(u, p)


def rk4_step(state, dt: float, op: MixedOperator, forcing=None, t: float = 0.0,
             step_index: int = 0) -> State:
    """Classical RK4 step of [u, p]' = Minv(-A[u, p] + f) (operator.py:506-531)
    on the device.  ``forcing(time) -> State`` is evaluated at t, t + dt/2
    and t + dt (the reference calls it at t + dt/2 for both middle stages)."""
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt}")
    try:
        if forcing is not None:
            return op.rk4_forced(state, dt, forcing(t), forcing(t + dt / 2), forcing(t + dt))
        return op.rk4(state, dt, 1)
    except DivergenceError as ex:
        raise DivergenceError(f"non-finite state after step {step_index}") from ex
