"""z-slab domain decomposition of the box mesh across ranks (host logic).

The reference is single-process (P = identity).  The paper's
multi-GPU P / P^T is the MPI group exchange of shared dofs.
Here rank r owns the contiguous element layers [z0, z1) (elements are
z-slowest, mesh.py:100) and therefore the contiguous global dof slice
[z0*p*npx*npy, (z1*p+1)*npx*npy) (dofs are z-slowest, mesh.py:164);
neighbouring slices overlap in exactly one npx*npy plane.

On the GPU the exchange lives inside libfk_b200 (fk_comm.cu: peer-memory
mailboxes over NVLink, or NCCL); the functions here are the same algorithm
on host tensors over any torch.distributed group, used by the gloo tests to
pin the partition math (tests/test_parallel.py) and by bench.py for rank
bookkeeping.  ``run_ranks`` drives an in-process (loopback) group: one host
thread and one CUDA stream per rank.
"""

from __future__ import annotations

import numpy as np


def slab_range(nz: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous element layers [z0, z1) of rank ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if nz < world:
        raise ValueError(f"{nz} element layers cannot be split over {world} ranks")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def plane_size(nx: int, ny: int, p: int) -> int:
    return (nx * p + 1) * (ny * p + 1)


def local_dof_range(nx: int, ny: int, p: int, z0: int, z1: int) -> tuple[int, int]:
    """Global ids [start, stop) of the dofs touched by layers [z0, z1)."""
    P = plane_size(nx, ny, p)
    return z0 * p * P, (z1 * p + 1) * P


def owned_range(nx: int, ny: int, p: int, z0: int, z1: int, rank: int) -> tuple[int, int]:
    """Global ids owned by ``rank`` (the lower rank owns each shared plane)."""
    start, stop = local_dof_range(nx, ny, p, z0, z1)
    if rank > 0:
        start += plane_size(nx, ny, p)
    return start, stop


def scatter_global(x: np.ndarray, nx, ny, p, z0, z1) -> np.ndarray:
    s, e = local_dof_range(nx, ny, p, z0, z1)
    return np.ascontiguousarray(x[s:e])


def exchange_planes(y_local, plane: int, rank: int, world: int, group=None):
    """In place: add the neighbours' partial sums of the shared planes
    (the host-tensor statement of fk_comm.cu:exchange_interface)."""
    import torch
    import torch.distributed as dist

    ops, recv = [], {}
    if rank > 0:
        recv["below"] = torch.empty(plane, dtype=y_local.dtype)
        ops.append(dist.P2POp(dist.isend, y_local[:plane].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv["below"], rank - 1, group))
    if rank < world - 1:
        recv["above"] = torch.empty(plane, dtype=y_local.dtype)
        ops.append(dist.P2POp(dist.isend, y_local[-plane:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv["above"], rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    if "below" in recv:
        y_local[:plane] += recv["below"]
    if "above" in recv:
        y_local[-plane:] += recv["above"]
    return y_local


def gather_global(y_local: np.ndarray, ndof_global: int, nx, ny, p, z0, z1, rank, group=None):
    """All-gather the owned parts of every rank into one global vector."""
    import torch
    import torch.distributed as dist

    s, e = owned_range(nx, ny, p, z0, z1, rank)
    ls, _ = local_dof_range(nx, ny, p, z0, z1)
    full = torch.zeros(ndof_global, dtype=torch.float64)
    full[s:e] = torch.as_tensor(np.asarray(y_local)[s - ls:e - ls])
    dist.all_reduce(full, group=group)
    return full.numpy()


def run_ranks(fn, nranks: int, streams=None, device=None):
    """Run ``fn(rank, stream, barrier)`` for every rank of an in-process group
    (``Comm.loopback``, one GPU per rank) on its own thread with its own CUDA
    stream current (the P2P exchange waits on the device for the peers, so
    ranks must be issued concurrently; allocate device memory before, not
    inside, ``fn`` — a device allocation may wait for a peer that is
    waiting for this rank).  Ranks sharing one GPU should be processes, not
    threads (see ``Comm``).
    Returns the list of results in rank order; re-raises the first
    exception."""
    import threading

    import torch

    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if streams is None:
        streams = [torch.cuda.Stream(device=dev) for _ in range(nranks)]
    bar = threading.Barrier(nranks)
    out, err = [None] * nranks, [None] * nranks

    def body(r):
        try:
            with torch.cuda.device(dev), torch.cuda.stream(streams[r]):
                out[r] = fn(r, streams[r], bar.wait)
                streams[r].synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e
            bar.abort()

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out
