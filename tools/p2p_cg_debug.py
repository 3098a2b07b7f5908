"""Loopback multi-rank CG probe with a mailbox-dumping watchdog.
    python tools/p2p_cg_debug.py WORLD DET ITERS"""
import ctypes, os, sys, threading, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09038_b200 import Comm, PAOperator, cg_solve, fem, parallel, _lib  # noqa: E402

world, det, iters = int(sys.argv[1]), bool(int(sys.argv[2])), int(sys.argv[3])
n, p = (3, 3, 8), 4
lib = _lib.load()
lib.fk_comm_debug_state.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]
for rep in range(2):
    comms = Comm.loopback(world, parallel.plane_size(n[0], n[1], p))
    streams = [torch.cuda.Stream() for _ in range(world)]
    ops = [PAOperator(fem.build_mesh(*n), p, dirichlet=True, deterministic=det, comm=comms[r],
                      stream=streams[r]) for r in range(world)]
    print("variants", [(o.variant, o.info.cfg) for o in ops], flush=True)
    rng = [parallel.local_dof_range(n[0], n[1], p, *comms[r].slab(n[2])) for r in range(world)]
    b = np.random.default_rng(5).standard_normal((n[0]*p+1)*(n[1]*p+1)*(n[2]*p+1))
    bs = [torch.as_tensor(b[s:e], device="cuda") for s, e in rng]
    xs = [torch.empty_like(v) for v in bs]
    torch.cuda.synchronize()
    done = threading.Event()

    def dump():
        for r, c in enumerate(comms):
            a = (ctypes.c_ulonglong * 8)()
            rc = lib.fk_comm_debug_state(c.handle, a)
            print(f"rank {r}: rc={rc} recv={a[0]},{a[1]} consumed={a[2]},{a[3]} seq_x={a[4]} seq_r={a[5]}", flush=True)

    def wd():
        if not done.wait(15):
            print("STALL rep", rep, flush=True); dump(); os._exit(3)
    threading.Thread(target=wd, daemon=True).start()
    t0 = time.time()
    hs = parallel.run_ranks(lambda r, s, bar: cg_solve(ops[r], bs[r], iters=iters, out=xs[r], barrier=bar)[1],
                            world, streams=streams)
    done.set()
    print("rep", rep, "ok", time.time() - t0, hs[0][-1], flush=True)
    dump()
    for o in ops: o.close()
    for c in comms: c.close()
