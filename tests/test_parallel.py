"""z-slab decomposition host logic on CPU with a world_size-2 gloo group.

The device path does the same exchange with NCCL inside libfk_b200
(fk_comm.cu); here the partition math, the interface-plane exchange and the
owned-dof dot products are pinned against the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bp
from paper_2603_09038_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_slab_ranges_cover_layers():
    for nz, world in [(96, 8), (54, 2), (7, 3), (5, 5)]:
        ranges = [parallel.slab_range(nz, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1
    with pytest.raises(ValueError):
        parallel.slab_range(3, 0, 4)


def test_local_and_owned_ranges_partition_global_dofs():
    nx, ny, nz, p = 3, 2, 7, 3
    ndof = bp.num_dofs(nx, ny, nz, p + 1)
    owned = []
    for world in (1, 2, 3, 7):
        owned = []
        for r in range(world):
            z0, z1 = parallel.slab_range(nz, r, world)
            s, e = parallel.local_dof_range(nx, ny, p, z0, z1)
            ids = bp.gather_ids(nx, ny, nz, p + 1, (z0, z1))
            assert ids.min() == s and ids.max() == e - 1  # no gaps
            owned.append(parallel.owned_range(nx, ny, p, z0, z1, r))
        cover = np.zeros(ndof, dtype=int)
        for s, e in owned:
            cover[s:e] += 1
        assert (cover == 1).all()


def _worker(rank, world, port, kind, n, p, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = n
        z0, z1 = parallel.slab_range(nz, rank, world)
        full = bp.Problem(kind, nx, ny, nz, p)
        slab = bp.Problem(kind, nx, ny, nz, p, ez_range=(z0, z1))
        x = np.random.default_rng(0).standard_normal(full.ndof)
        s, e = parallel.local_dof_range(nx, ny, p, z0, z1)
        # element-local apply of this rank's slab, in slab-local numbering
        xe = x[slab.ids]
        ye = slab.element_apply(xe)
        y_local = bp.scatter_add(slab.ids - s, ye, e - s)
        y_t = torch.as_tensor(y_local)
        parallel.exchange_planes(y_t, parallel.plane_size(nx, ny, p), rank, world)
        y_ref = full.apply(x)[s:e]
        err = float(np.max(np.abs(y_t.numpy() - y_ref)) / np.max(np.abs(y_ref)))
        # owned-dof dot product == global dot product
        os_, oe = parallel.owned_range(nx, ny, p, z0, z1, rank)
        d = torch.tensor([float(x[os_:oe] @ y_t.numpy()[os_ - s:oe - s])], dtype=torch.float64)
        dist.all_reduce(d)
        gdot = float(x @ full.apply(x))
        yg = parallel.gather_global(y_t.numpy(), full.ndof, nx, ny, p, z0, z1, rank)
        gerr = float(np.max(np.abs(yg - full.apply(x))))
        out[rank] = (err, abs(float(d) - gdot) / abs(gdot), gerr)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,p,world", [("diffusion", (3, 2, 4), 3, 2), ("mass", (2, 3, 5), 2, 2),
                                             ("diffusion", (2, 2, 6), 4, 3)])
def test_slab_exchange_matches_single_process(kind, n, p, world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, kind, n, p, out), nprocs=world, join=True,
                       start_method="fork")
    for r in range(world):
        err, dot_err, gerr = out[r]
        assert err <= 1e-14  # normwise vs single process (summation order differs)
        assert dot_err <= 1e-13
        assert gerr <= 1e-13


def test_bench_spawn_translates_n_for_torchrun(monkeypatch):
    """bench.py --gpus N without torchrun re-launches itself under
    torch.distributed.run; torchrun's parser would take '--n' as an
    abbreviation of its own options, so it is passed as '--elems'."""
    import importlib.util
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}
    monkeypatch.setattr(subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr("sys.argv", ["bench.py", "--gpus", "4", "--n", "24", "--steps", "3"])
    a = bench.parse()
    assert a.n == 24 and a.gpus == 4
    bench.spawn_ranks(a)
    cmd = seen["cmd"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    tail = cmd[cmd.index(os.path.abspath(os.path.join(root, "bench.py"))) + 1:]
    assert tail == ["--gpus", "4", "--elems", "24", "--steps", "3"]
