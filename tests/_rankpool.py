"""A persistent group of rank PROCESSES sharing one GPU, for the multi-rank tests.

Every rank is its own process with its own CUDA context — the deployment
topology of an 8-GPU box (one process per GPU, mailboxes mapped with CUDA
IPC, bootstrap over torch.distributed/gloo), except that here all ranks sit
on cuda:0.  Contexts of different processes are time-sliced with compute
preemption, so a rank whose exchange kernel waits for a peer always yields
the GPU to that peer; ranks driven by threads of ONE process have no such
guarantee (kernels of different streams may share a hardware queue).

    pool = RankPool(3)
    results = pool.run("apply", kind="diffusion", n=(3, 2, 6), p=4)   # list, rank order
    pool.close()

Tasks are the functions ``task_<name>(rank, world, **kw)`` of
tests/_rank_tasks.py; they build their own communicator and operators and
return picklable results (NumPy arrays).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import socket
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _worker(rank, world, port, conn):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist

        import _rank_tasks

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        conn.send(("ready", None))
    except BaseException:  # noqa: BLE001 - reported to the parent
        conn.send(("error", traceback.format_exc()))
        return
    while True:
        msg = conn.recv()
        if msg is None:
            break
        name, kw = msg
        try:
            res = getattr(_rank_tasks, f"task_{name}")(rank, world, **kw)
            conn.send(("ok", res))
        except BaseException:  # noqa: BLE001
            conn.send(("error", traceback.format_exc()))
    dist.destroy_process_group()


class RankPool:
    def __init__(self, world: int, timeout: float = 240.0):
        ctx = mp.get_context("spawn")
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        self.world, self.timeout = world, timeout
        self.conns, self.procs = [], []
        for r in range(world):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(r, world, port, b), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for r, c in enumerate(self.conns):
            self._recv(r, c)

    def _recv(self, r, c):
        if not c.poll(self.timeout):
            self.close(kill=True)
            raise TimeoutError(f"rank {r} did not answer within {self.timeout} s")
        status, val = c.recv()
        if status == "error":
            self.close(kill=True)
            raise RuntimeError(f"rank {r} failed:\n{val}")
        return val

    def run(self, name: str, **kw):
        for c in self.conns:
            c.send((name, kw))
        return [self._recv(r, c) for r, c in enumerate(self.conns)]

    def close(self, kill: bool = False):
        for c, p in zip(self.conns, self.procs):
            if not kill and p.is_alive():
                try:
                    c.send(None)
                except Exception:
                    pass
        for p in self.procs:
            p.join(timeout=0 if kill else 20)
            if p.is_alive():
                p.kill()
                p.join()
        self.procs, self.conns = [], []
