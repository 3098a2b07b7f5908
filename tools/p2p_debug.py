"""Loopback P2P exchange probe: N ranks on one GPU, one thread + stream each,
a watchdog prints every rank's mailbox control words if the group stalls.
    python tools/p2p_debug.py WORLD NZ REPS [--legacy-sync]
"""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09038_b200 import Comm, PAOperator, fem, parallel, _lib  # noqa: E402

world, nz, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n, p = (3, 2, nz), 3
lib = _lib.load()
lib.fk_comm_debug_state.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]
comms = Comm.loopback(world, parallel.plane_size(n[0], n[1], p))
streams = [torch.cuda.Stream() for _ in range(world)]
print("streams", [s.cuda_stream for s in streams], flush=True)
ops = [PAOperator(fem.build_mesh(*n), p, comm=comms[r], stream=streams[r]) for r in range(world)]
xs = [torch.randn(op.num_dofs, dtype=torch.float64, device="cuda") for op in ops]
ys = [torch.empty_like(x) for x in xs]
torch.cuda.synchronize()
done = threading.Event()


def dump():
    for r, c in enumerate(comms):
        a = (ctypes.c_ulonglong * 8)()
        rc = lib.fk_comm_debug_state(c.handle, a)
        print(f"rank {r}: rc={rc} recv={a[0]},{a[1]} consumed={a[2]},{a[3]} seq_x={a[4]} seq_r={a[5]} "
              f"put_done={a[6]} add_done={a[7]}", flush=True)


def watchdog():
    if not done.wait(8):
        print("STALL", flush=True)
        dump()
        os._exit(3)


threading.Thread(target=watchdog, daemon=True).start()
t0 = time.time()
parallel.run_ranks(lambda r, s, bar: [ops[r].apply(xs[r], out=ys[r]) for _ in range(reps)], world,
                   streams=streams)
done.set()
print(f"ok world={world} nz={nz} reps={reps} {time.time() - t0:.3f}s", flush=True)
dump()
