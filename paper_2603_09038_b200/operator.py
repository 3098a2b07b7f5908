"""PA operator (CEED BP1 mass / BP3 diffusion) and Jacobi-PCG on B200.

Drop-in sibling of the reference operator API (feklab/operator.py):

* ``setup_pa_data``  ~ ``setup_quad_data`` (operator.py:147-193): host-side PA
  quadrature data, in the exact arithmetic the device setup kernel uses.
* ``PAOperator``     ~ ``BlockOperator`` (operator.py:221-362): built from a
  mesh and order (or the reference's own ``Mesh``/``Basis1D``/``Restriction``
  objects), ``.apply(x)`` validates the vector length exactly like
  ``BlockOperator.apply`` (ValueError "... do not match ...",
  operator.py:333-338), bumps ``counters.operator_applies`` and the analytic
  flop / D-read counts (counters.py:8-29), then runs the fused sm_100a kernel.
* ``cg_solve``       Jacobi-PCG with MFEM CGSolver semantics (not in the
  reference), device-resident, graph-replayed.

``x`` may be a CUDA float64 torch tensor (result stays on the device) or a
NumPy array (host buffers: copied in, applied, copied out).  There is no CPU
fallback: constructing an operator without the CUDA library or a GPU raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fem import Basis1D, Counters, ShapeError

# PA / FusedPA: stored quadrature data (one fused kernel either way for a
# single-block operator); MF / FusedMF: the factors recomputed in the kernel
# (operator.py:16-19, 280-286) -> variant "mf"
STRATEGIES = ("PA", "FusedPA", "MF", "FusedMF")
KINDS = {"mass": _lib.FK_KIND_MASS, "diffusion": _lib.FK_KIND_DIFFUSION,
         "bp1": _lib.FK_KIND_MASS, "bp3": _lib.FK_KIND_DIFFUSION}


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# host-side PA data (setup_quad_data analogue)
# ---------------------------------------------------------------------------


@dataclass
class PAData:
    """PA quadrature data of one element (identical for every element of the
    axis-aligned box): ``d[comp, qp]`` with qp = a + q*(b + q*c).

    BP1: one component, w_a w_b w_c |J|.  BP3: the six components
    (00, 01, 02, 11, 12, 22) of w|J| J^-1 J^-T (operator.py:137-144 gives the
    one-sided w|J| J^-1; the diffusion data is its symmetric square)."""

    kind: str
    d: np.ndarray
    num_elements: int

    @property
    def ncomp(self) -> int:
        return self.d.shape[0]


def setup_pa_data(mesh, basis, kind: str = "diffusion") -> PAData:
    w = np.asarray(basis.quad_weights, dtype=np.float64)
    wdet = np.kron(w, np.kron(w, w)) * mesh.jacobian_det  # operator.py:132-134, :171
    if KINDS[kind] == _lib.FK_KIND_MASS:
        return PAData("mass", wdet[None, :].copy(), mesh.num_elements)
    jinv = 1.0 / np.asarray(mesh.jacobian_diag, dtype=np.float64)
    z = np.zeros_like(wdet)
    d = np.stack([wdet * (jinv[0] * jinv[0]), z, z, wdet * (jinv[1] * jinv[1]), z,
                  wdet * (jinv[2] * jinv[2])])
    return PAData("diffusion", d, mesh.num_elements)


def flops_per_element(kind: str, d: int, q: int) -> int:
    """Algorithmic flops of the stage-shared apply."""
    if KINDS[kind] == _lib.FK_KIND_MASS:
        return 4 * (q * d ** 3 + q * q * d * d + q ** 3 * d) + q ** 3
    return 2 * (4 * q * d ** 3 + 6 * q * q * d * d + 6 * q ** 3 * d) + 15 * q ** 3


def bytes_per_apply(kind: str, ndof: int, nel: int, d: int, q: int, mf: bool = False) -> int:
    """Algorithmic HBM bytes: x read, y write, D (not for the
    matrix-free variant), int32 map."""
    ncomp = 0 if mf else (1 if KINDS[kind] == _lib.FK_KIND_MASS else 6)
    return 16 * ndof + 8 * ncomp * q ** 3 * nel + 4 * d ** 3 * nel


# ---------------------------------------------------------------------------
# operator
# ---------------------------------------------------------------------------


class PAOperator:
    """Matrix-free PA operator y = A x for BP1 (kind="mass") or BP3
    (kind="diffusion") on an nx*ny*nz box of order-p hexahedra.

    Parameters mirror BlockOperator (operator.py:224-239): ``mesh`` is any
    object with nx, ny, nz, jacobian_diag, jacobian_det (feklab.mesh.Mesh or
    paper_2603_09038_b200.fem.Mesh); ``basis`` defaults to
    Basis1D.nodal(order+1, num_quad_1d) and may be the reference's Basis1D;
    ``restriction`` (optional) is a Restriction whose gather_ids the device
    map is built from instead of the closed form.  ``deterministic=True`` is
    the verification mode: elements run in 8-colour order with one launch
    per colour, so every dof sums its contributions in a fixed order and
    apply / diagonal / cg_solve are bitwise reproducible run to run (the
    reference's np.add.at scatter is sequential, mesh.py:133-137).
    """

    def __init__(self, mesh, order: int, num_quad_1d: int | None = None,
                 kind: str = "diffusion", strategy: str = "FusedPA",
                 dirichlet: bool = False, counters: Counters | None = None,
                 device=None, basis=None, restriction=None, variant: str = "auto",
                 comm: "Comm | None" = None, z_range: tuple[int, int] | None = None,
                 stream=None, deterministic: bool = False):
        if kind not in KINDS:
            raise ValueError(f"kind must be one of {tuple(KINDS)}, got {kind!r}")
        if strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
        if variant not in _lib.VARIANTS:
            raise ValueError(f"variant must be one of {tuple(_lib.VARIANTS)}, got {variant!r}")
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("PAOperator needs a CUDA device (there is no CPU fallback)")
        lib = _lib.load()
        self.kind = "mass" if KINDS[kind] == _lib.FK_KIND_MASS else "diffusion"
        self.strategy = strategy
        if strategy in ("MF", "FusedMF"):
            if variant not in ("auto", "mf"):
                raise ValueError(f"strategy {strategy!r} runs the matrix-free variant, got {variant!r}")
            variant = "mf"
        self.mesh = mesh
        self.order = int(order)
        q = int(num_quad_1d) if num_quad_1d is not None else self.order + 2
        self.basis = basis if basis is not None else Basis1D.nodal(self.order + 1, q)
        if self.basis.num_dofs_1d != self.order + 1 or self.basis.num_quad_1d != q:
            raise ShapeError(
                f"basis ({self.basis.num_dofs_1d}, {self.basis.num_quad_1d}) does not match "
                f"order {self.order} / num_quad_1d {q}")
        self.num_quad_1d = q
        self.dirichlet = bool(dirichlet)
        self.counters = counters if counters is not None else Counters()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.comm = comm
        nz = mesh.nz
        z0, z1 = (0, nz) if z_range is None else (int(z_range[0]), int(z_range[1]))
        if comm is not None and z_range is None:
            z0, z1 = comm.slab(nz)
        self.z_range = (z0, z1)
        with torch.cuda.device(self.device):
            self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._B = np.ascontiguousarray(self.basis.values, dtype=np.float64)
        self._G = np.ascontiguousarray(self.basis.gradients, dtype=np.float64)
        self._w = np.ascontiguousarray(self.basis.quad_weights, dtype=np.float64)
        desc = _lib.FkOpDesc()
        desc.kind = KINDS[kind]
        desc.p = self.order
        desc.q = q
        desc.nx, desc.ny = mesh.nx, mesh.ny
        desc.nz_local, desc.z0_layer, desc.nz_global = z1 - z0, z0, nz
        jd = np.asarray(mesh.jacobian_diag, dtype=np.float64)
        for s in range(3):
            desc.jac_diag[s] = float(jd[s])
        desc.jac_det = float(mesh.jacobian_det)
        dp = ctypes.POINTER(ctypes.c_double)
        desc.B = self._B.ctypes.data_as(dp)
        desc.G = self._G.ctypes.data_as(dp)
        desc.w = self._w.ctypes.data_as(dp)
        self._gids_host = None
        if restriction is not None:
            ids = np.ascontiguousarray(restriction.gather_ids, dtype=np.int64)
            nxy = mesh.nx * mesh.ny
            ids = np.ascontiguousarray(ids[z0 * nxy: z1 * nxy])
            d3 = (self.order + 1) ** 3
            if ids.shape != ((z1 - z0) * nxy, d3):
                raise ValueError(f"restriction {ids.shape} does not match mesh/order "
                                 f"({(z1 - z0) * nxy}, {d3})")
            self._gids_host = ids
            desc.gather_ids = ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        desc.dirichlet = 1 if self.dirichlet else 0
        # verification mode: colour-ordered elements, bitwise reproducible
        # y, diagonal and CG (fk.h fk_op_desc.deterministic)
        self.deterministic = bool(deterministic)
        desc.deterministic = 1 if self.deterministic else 0
        desc.variant = _lib.VARIANTS[variant]
        desc.device = self.device.index
        desc.stream = ctypes.c_void_p(self._stream.cuda_stream)
        if comm is not None:
            comm.attach((mesh.nx * self.order + 1) * (mesh.ny * self.order + 1))
        desc.comm = comm.handle if comm is not None else None
        self._lib = lib
        h = ctypes.c_void_p()
        _lib.check(lib.fk_op_create(ctypes.byref(h), ctypes.byref(desc)))
        self._h = h
        _lib.check(lib.fk_op_setup(self._h))
        self.info = self._info()
        self.num_dofs = int(self.info.ndof_local)
        self.num_elements = int(self.info.nel_local)
        self.dof_offset = int(self.info.dof_offset)
        self.num_global_dofs = int(self.info.ndof_global)
        d, qq = self.order + 1, q
        self.flops_per_apply = flops_per_element(self.kind, d, qq) * self.num_elements
        self._bytes = {mf: bytes_per_apply(self.kind, self.num_dofs, self.num_elements, d, qq, mf)
                       for mf in (False, True)}
        self._ncomp = 1 if self.kind == "mass" else 6

    @property
    def bytes_per_apply(self) -> int:
        """Algorithmic HBM bytes of one apply with the current variant."""
        return self._bytes[self.variant == "mf"]

    # -- lifecycle ------------------------------------------------------------

    def _info(self) -> _lib.FkOpInfo:
        info = _lib.FkOpInfo()
        _lib.check(self._lib.fk_op_get_info(self._h, ctypes.byref(info)))
        return info

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.fk_op_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def variant(self) -> str:
        return _lib.VARIANT_NAMES[self.info.variant]

    def set_variant(self, variant: str) -> None:
        if variant not in _lib.VARIANTS:
            raise ValueError(f"variant must be one of {tuple(_lib.VARIANTS)}, got {variant!r}")
        _lib.check(self._lib.fk_op_set_variant(self._h, _lib.VARIANTS[variant]))
        self.info = self._info()

    def set_config(self, variant: str, cfg: int) -> None:
        """Pick compiled launch geometry ``cfg`` of ``variant`` ("dfma"/"dmma")."""
        if variant not in ("dfma", "dmma", "eo", "mf"):
            raise ValueError(f"variant must be 'dfma', 'dmma', 'eo' or 'mf', got {variant!r}")
        _lib.check(self._lib.fk_op_set_config(self._h, _lib.VARIANTS[variant], int(cfg)))
        self.info = self._info()

    @property
    def launch(self) -> tuple[int, int, int]:
        """(elements per CTA, threads per CTA, persistent CTAs)."""
        i = self._info()
        return i.elems_per_block, i.threads_per_block, i.blocks

    # -- vectors --------------------------------------------------------------

    def zeros(self):
        torch = _torch()
        return torch.zeros(self.num_dofs, dtype=torch.float64, device=self.device)

    def _check_vec(self, v, name="vector"):
        n = v.shape[0] if v.ndim == 1 else None
        if v.ndim != 1 or n != self.num_dofs:
            raise ValueError(f"{name} dimensions {tuple(v.shape)} do not match operator "
                             f"({self.num_dofs},)")

    def _dev(self, v, name="vector"):
        torch = _torch()
        if not isinstance(v, torch.Tensor) or not v.is_cuda:
            raise TypeError(f"{name} must be a CUDA tensor")
        self._check_vec(v, name)
        if v.dtype != torch.float64 or not v.is_contiguous() or v.device != self.device:
            raise ValueError(f"{name} must be a contiguous float64 tensor on {self.device}")
        return v

    def _host(self, v, name="vector"):
        """A host buffer the C side may read/write num_dofs doubles through:
        C-contiguous float64 NumPy array or CPU torch tensor of exactly that
        length (anything else would overrun or corrupt memory)."""
        torch = _torch()
        if isinstance(v, torch.Tensor):
            if v.is_cuda or v.dtype != torch.float64 or not v.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float64 CPU tensor")
            self._check_vec(v, name)
            return v.data_ptr()
        if not isinstance(v, np.ndarray):
            raise TypeError(f"{name} must be a NumPy array or a CPU torch tensor")
        if v.dtype != np.float64 or not v.flags.c_contiguous:
            raise ValueError(f"{name} must be a C-contiguous float64 array")
        self._check_vec(v, name)
        return v.ctypes.data

    def _count(self, n: int = 1) -> None:
        """Reference counter semantics (counters.py:8-29, operator.py:280-286):
        every apply bumps operator_applies and the flops; only the PA
        strategies read stored quadrature data, the matrix-free ones count
        no d_reads."""
        self.counters.operator_applies += n
        self.counters.flops += n * self.flops_per_apply
        if self.variant != "mf":
            self.counters.d_reads += n * self._ncomp * self.num_quad_1d ** 3 * self.num_elements

    # -- apply ----------------------------------------------------------------

    def apply(self, x, out=None):
        """y = A x (assembled over ranks, Dirichlet-constrained if requested)."""
        torch = _torch()
        if isinstance(x, np.ndarray):
            xh = np.ascontiguousarray(x, dtype=np.float64)
            self._check_vec(xh, "state")
            yh = np.empty_like(xh) if out is None else out
            yp = self._host(yh, "out")
            self._count()
            _lib.check(self._lib.fk_op_apply_host(self._h, xh.ctypes.data, yp))
            return yh
        x = self._dev(x, "state")
        y = torch.empty_like(x) if out is None else self._dev(out, "out")
        if y.data_ptr() == x.data_ptr():
            raise ValueError("in-place apply (out is x) is not supported")
        self._count()
        _lib.check(self._lib.fk_op_apply(self._h, x.data_ptr(), y.data_ptr()))
        return y

    mult = apply
    __call__ = apply

    def apply_host(self, x: np.ndarray, out: np.ndarray) -> np.ndarray:
        """Host-buffer apply without allocation (pinned ``x``/``out`` give full PCIe speed)."""
        xp, yp = self._host(x, "x"), self._host(out, "out")
        self._count()
        _lib.check(self._lib.fk_op_apply_host(self._h, xp, yp))
        return out

    def apply_local(self, x, out=None):
        """Element-local G^T A_E G x without interface exchange or Dirichlet."""
        torch = _torch()
        x = self._dev(x, "state")
        y = torch.empty_like(x) if out is None else self._dev(out, "out")
        self._count()
        _lib.check(self._lib.fk_op_apply_local(self._h, x.data_ptr(), y.data_ptr()))
        return y

    def diagonal(self, out=None):
        d = self.zeros() if out is None else self._dev(out, "out")
        _lib.check(self._lib.fk_op_diagonal(self._h, d.data_ptr()))
        return d

    def set_essential(self, v, value: float = 0.0):
        """v[ess] = value on this rank's Dirichlet dofs (in place)."""
        self._dev(v, "v")
        _lib.check(self._lib.fk_op_set_essential(self._h, v.data_ptr(), float(value)))
        return v

    def prepare_cg(self, iters: int) -> None:
        """Allocate the CG workspace now (fk_cg_prepare)."""
        _lib.check(self._lib.fk_cg_prepare(self._h, int(iters)))

    def dot(self, a, b) -> float:
        """Global (all-rank) dot product over owned dofs."""
        self._dev(a, "a")
        self._dev(b, "b")
        out = ctypes.c_double()
        _lib.check(self._lib.fk_dot(self._h, a.data_ptr(), b.data_ptr(), ctypes.byref(out)))
        return out.value

    # -- parity hooks -----------------------------------------------------------

    def restriction_ids(self) -> np.ndarray:
        d3 = (self.order + 1) ** 3
        out = np.empty((self.num_elements, d3), dtype=np.int64)
        _lib.check(self._lib.fk_op_restriction(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out

    def pa_data(self) -> np.ndarray:
        q3 = self.num_quad_1d ** 3
        out = np.empty((self.num_elements, self._ncomp, q3), dtype=np.float64)
        _lib.check(self._lib.fk_op_pa_data(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    # -- timing (bench) -----------------------------------------------------------

    def time_apply(self, x, y, reps: int, flush=None) -> tuple[float, float]:
        """Mean (ms per full apply, ms of the fused kernel) over ``reps`` applies,
        CUDA events on the operator's stream; ``flush`` (a CUDA tensor) is
        overwritten before each apply (untimed) to evict L2."""
        fa, fk = ctypes.c_double(), ctypes.c_double()
        fptr = flush.data_ptr() if flush is not None else None
        fbytes = flush.numel() * flush.element_size() if flush is not None else 0
        self._count(reps)
        _lib.check(self._lib.fk_op_time_apply(self._h, x.data_ptr(), y.data_ptr(), int(reps),
                                              fptr, fbytes, ctypes.byref(fa), ctypes.byref(fk)))
        return fa.value, fk.value


# ---------------------------------------------------------------------------
# CG
# ---------------------------------------------------------------------------


def cg_solve(op: PAOperator, b, iters: int = 100, rtol: float = 0.0, out=None, barrier=None):
    """Jacobi-PCG on ``op`` (build it with dirichlet=True for BP3), x0 = 0.

    Returns (x, history) with history[k] = sqrt(r_k . z_k), k = 0..iters_done.
    ``b`` may be a NumPy array (x returned as NumPy) or a CUDA tensor; ``out``
    an optional preallocated CUDA solution vector.  ``barrier`` (callable) is
    run after the workspace is allocated and before the solve starts — ranks
    of a loopback group on one GPU pass a shared barrier so that no rank
    allocates device memory while a peer waits on the device.
    """
    torch = _torch()
    host = isinstance(b, np.ndarray)
    bd = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64), device=op.device) if host else op._dev(b, "b")
    if host:
        op._check_vec(bd, "b")
    x = torch.empty_like(bd) if out is None else op._dev(out, "x")
    hist = np.zeros(iters + 1)
    done = ctypes.c_int()
    _lib.check(op._lib.fk_cg_prepare(op._h, int(iters)))
    if barrier is not None:
        barrier()
    _lib.check(op._lib.fk_cg_solve(op._h, bd.data_ptr(), x.data_ptr(), int(iters), float(rtol),
                                   hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   ctypes.byref(done)))
    op._count(done.value)  # applies actually run (rtol may stop early)
    hist = hist[: done.value + 1]
    return (x.cpu().numpy() if host else x), hist


# ---------------------------------------------------------------------------
# multi-GPU communicator
# ---------------------------------------------------------------------------


class Comm:
    """One z-slab communicator per rank.

    ``transport="p2p"`` (default): the peer-memory transport of fk_comm.cu —
    each rank's mailbox is mapped into its peers with CUDA IPC (handles
    all-gathered over ``group``, any torch.distributed backend), halo planes
    and CG scalars move by NVLink stores with device-side flags.  The mailbox
    is sized for interface planes of ``plane_cap`` doubles; with
    ``plane_cap=None`` it is created by the first operator attached (every
    rank attaches collectively, as it constructs its operator).
    ``transport="nccl"``: grouped ncclSend/ncclRecv + ncclAllReduce; the
    128-byte ncclUniqueId is produced by rank 0 and broadcast over ``group``.
    If the CUDA-IPC mapping fails on any rank (no peer access on some pair),
    all ranks agree and fall back to NCCL (``fallback=False``: raise).

    ``Comm.loopback(n, plane_cap, devices)`` builds n ranks inside this
    process, one per GPU; drive each rank from its own thread and stream
    (``parallel.run_ranks``).  Ranks that share ONE GPU belong in separate
    processes (CUDA-IPC path above): kernels of different streams of one
    process are not guaranteed to run concurrently (streams may share a
    hardware queue), so a rank waiting on the device for a peer in the same
    process can stall; contexts of different processes are time-sliced with
    preemption and always progress (tests/_rankpool.py)."""

    def __init__(self, rank: int, world_size: int, device: int, group=None,
                 transport: str = "p2p", plane_cap: int | None = None, fallback: bool = True):
        if transport not in _lib.TRANSPORTS:
            raise ValueError(f"transport must be one of {tuple(_lib.TRANSPORTS)}, got {transport!r}")
        if not 0 <= rank < world_size:
            raise ValueError(f"bad rank {rank} of {world_size}")
        self._lib = _lib.load()
        self.rank, self.world_size, self.device = rank, world_size, device
        self.transport = transport
        self.group = group
        self.fallback = bool(fallback)
        self.handle = None
        self.plane_cap = None
        if transport == "nccl":
            self._create_nccl()
        elif plane_cap is not None:
            self._create_p2p(int(plane_cap))

    def _create_p2p(self, plane_cap: int) -> None:
        h = ctypes.c_void_p()
        mine = (ctypes.c_char * _lib.FK_IPC_HANDLE_BYTES)()
        _lib.check(self._lib.fk_comm_create_p2p(ctypes.byref(h), self.rank, self.world_size,
                                                self.device, int(plane_cap), mine))
        self.handle, self.plane_cap = h, int(plane_cap)
        if self.world_size > 1:
            import torch.distributed as dist

            handles = [None] * self.world_size
            dist.all_gather_object(handles, bytes(mine), group=self.group)
            blob = (ctypes.c_char * (_lib.FK_IPC_HANDLE_BYTES * self.world_size)).from_buffer_copy(
                b"".join(handles))
            rc = self._lib.fk_comm_connect_p2p(self.handle, blob)
            err = self._lib.fk_last_error().decode(errors="replace") if rc else ""
            # agree on the outcome: a node without peer access on some pair
            # falls back to NCCL on every rank together
            oks = [None] * self.world_size
            dist.all_gather_object(oks, rc == _lib.FK_OK, group=self.group)
            if not all(oks):
                self._lib.fk_comm_destroy(self.handle)
                self.handle = None
                if not self.fallback:
                    raise _lib.FkError(_lib.FK_ECUDA, f"P2P mailboxes could not be mapped: {err}")
                import warnings

                warnings.warn(f"rank {self.rank}: CUDA-IPC peer mapping failed ({err or 'on a peer'}); "
                              "falling back to the NCCL transport")
                self.transport = "nccl"
                self._create_nccl()
                return
            # every rank's mappings exist before any rank stores into a peer
            dist.barrier(group=self.group)

    def _create_nccl(self) -> None:
        import torch.distributed as dist

        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            _lib.check(self._lib.fk_comm_unique_id(uid))
        payload = [bytes(uid)]
        if self.world_size > 1:
            dist.broadcast_object_list(payload, src=0, group=self.group)
        uid = (ctypes.c_char * 128).from_buffer_copy(payload[0])
        h = ctypes.c_void_p()
        _lib.check(self._lib.fk_comm_create(ctypes.byref(h), uid, self.rank, self.world_size,
                                            self.device))
        self.handle = h

    @classmethod
    def loopback(cls, nranks: int, plane_cap: int, devices=None) -> list["Comm"]:
        """``nranks`` P2P communicators in this process (rank r on devices[r],
        default all on the current device)."""
        lib = _lib.load()
        if devices is None:
            import torch

            devices = [torch.cuda.current_device()] * nranks
        if len(devices) != nranks:
            raise ValueError(f"{len(devices)} devices do not match {nranks} ranks")
        hs = (ctypes.c_void_p * nranks)()
        devs = (ctypes.c_int * nranks)(*[int(d) for d in devices])
        _lib.check(lib.fk_comm_create_loopback(hs, nranks, devs, int(plane_cap)))
        out = []
        for r in range(nranks):
            c = cls.__new__(cls)
            c._lib, c.rank, c.world_size, c.device = lib, r, nranks, int(devices[r])
            c.transport, c.group, c.plane_cap = "p2p", None, int(plane_cap)
            c.handle = ctypes.c_void_p(hs[r])
            out.append(c)
        return out

    def attach(self, plane: int) -> None:
        """Called by an operator with interface planes of ``plane`` dofs."""
        if self.transport != "p2p":
            return
        if self.handle is None:
            self._create_p2p(plane)
        elif plane > self.plane_cap:
            raise ValueError(f"interface plane of {plane} dofs does not match the communicator's "
                             f"capacity ({self.plane_cap})")

    def slab(self, nz: int) -> tuple[int, int]:
        from .parallel import slab_range

        return slab_range(nz, self.rank, self.world_size)

    def close(self):
        if self.handle is not None and self.handle.value:
            self._lib.fk_comm_destroy(self.handle)
        self.handle = None
