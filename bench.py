#!/usr/bin/env python
"""Benchmark: GDOF/s of the PA operator apply (BP3 diffusion) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--p 4] [--n 54] [--variant auto|dfma|dmma] [--sweep FILE]

A step is one operator apply y = A x (gather, B/G contractions, PA data D,
transposed contractions, scatter-add, and for N>1 the NCCL interface
exchange) over the whole mesh, inputs resident in HBM.  Default workload =
BASELINE.json configs[1]: BP3, p=4, q=6, 54^3 elements (10,218,313 dofs).
For N>1 (torchrun) every rank owns a 54^3-element z-slab of a 54x54x(54N)
mesh (weak scaling) and the slabs exchange their interface planes.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
CPU algorithm (the oracle/ restatement, per-element NumPy path exactly as
feklab executes it) over all host cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDOF/s of PA operator apply (BP3 diffusion, p=1..8) at 1/2/4/8 B200"
UNIT = "GDOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="diffusion", choices=["diffusion", "mass"])
    ap.add_argument("--p", type=int, default=None, help="order (default 4; 6 for --cg strong)")
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--n", type=int, default=None, help="elements per direction (per-rank slab is n^3)")
    ap.add_argument("--variant", default="auto", choices=["auto", "dfma", "dmma", "eo", "mf"])
    ap.add_argument("--sweep", default=None, help="also run the p=1..8 DFMA/DMMA sweep, JSON lines to FILE")
    ap.add_argument("--sweep-cfgs", default=None,
                    help="restrict the sweep to these geometries, e.g. 'eo0,eo9,dfma2'")
    ap.add_argument("--sweep-kinds", default="diffusion,mass")
    ap.add_argument("--sweep-orders", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--cg", default=None, choices=["weak", "strong"],
                    help="run the 100-iteration Jacobi-PCG benchmark (BASELINE configs[3]/[4])")
    ap.add_argument("--mixed", action="store_true",
                    help="acoustic-gravity FusedPA block apply (paper Table VII: H1 p=4 x L2 p=3, "
                         "q=5, ~540 M dofs; SURVEY.md §8f) + an RK4 step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


# sweep meshes: ~10 M dofs per order
SWEEP_N = {1: 214, 2: 107, 3: 71, 4: 54, 5: 43, 6: 36, 7: 31, 8: 27}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kind, p, n):
    """dram bytes per launch of the fused kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(f"{kind}_p{p}_n{n}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi needs a moment to start: wait (bounded) for its first
            # sample so the (short) timed region that follows is covered
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def count(self) -> int:
        return len(self.lines)

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle = restatement of the reference's per-element NumPy path)
# ---------------------------------------------------------------------------


_CPU = {}


def _cpu_worker(args):
    kind, n, p, q, e0, e1, reps = args
    from oracle import bp

    P, x = _CPU["problem"], _CPU["x"]  # inherited from the parent via fork
    ids = bp.gather_ids_elements(n, n, n, p + 1, e0, e1)
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        xe = x[ids]
        ye = P.element_apply(xe, batched=False)
        y = np.zeros(P.ndof)
        np.add.at(y, ids.ravel(), ye.ravel())
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return e1 - e0, best


def cpu_baseline(kind, n, p, q, seconds, cores=None):
    """Time the reference algorithm on a bounded contiguous element sample over
    all host cores; extrapolate GDOF/s by the sample's share of the elements."""
    import multiprocessing as mp

    from oracle import bp

    cores = cores or os.cpu_count() or 1
    P = bp.Problem(kind, 2, 2, 2, p, q)
    _CPU["problem"] = P  # element operator only depends on (p, q, h): use h of the n^3 mesh
    P.jd, P.detj = bp.jacobian(n, n, n)
    P.jinv = 1.0 / P.jd
    P.wdet = bp.quad_weights_3d(P.w) * P.detj
    P.ndof = bp.num_dofs(n, n, n, P.d)
    _CPU["x"] = np.random.default_rng(0).standard_normal(P.ndof)
    xe = np.random.default_rng(0).standard_normal((8, P.d ** 3))
    P.element_apply(xe, batched=False)
    t = time.perf_counter()
    P.element_apply(np.repeat(xe, 4, axis=0), batched=False)
    per_el = (time.perf_counter() - t) / 32
    per_worker = max(4, int(seconds / max(per_el, 1e-6) / 2))
    nel = n ** 3
    per_worker = min(per_worker, max(1, nel // cores))
    jobs = [(kind, n, p, q, w * per_worker, (w + 1) * per_worker, 2) for w in range(cores)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    sample_el = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    ndof = (n * p + 1) ** 3
    dofs = ndof * sample_el / nel
    return {"value": dofs / slowest / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{sample_el} of {nel} elements ({kind} p={p} {n}^3), per-element NumPy "
                      f"restatement of feklab's path, {cores} processes, best of 2, "
                      f"throughput scaled by element share; wall {wall:.1f}s"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = a.p or 4
    q = a.q or p + 2
    n = a.n or SWEEP_N.get(p, 54)
    budget = max(1.0, min(5.0, 150.0 / max(1, a.steps + a.warmup)))
    for _ in range(a.warmup):
        cpu_baseline(a.kind, n, p, q, budget * 0.25)
    vals = [cpu_baseline(a.kind, n, p, q, budget) for _ in range(max(1, min(a.steps, 5)))]
    v = statistics.median(r["value"] for r in vals)
    ndof = (n * p + 1) ** 3
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ndof / (v * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (x ~ N(0,1), seed 0)",
        "config": {"workload": f"BP3 PA diffusion apply p={p} q={q} {n}^3 ({ndof} dofs)" if a.kind == "diffusion"
                   else f"BP1 PA mass apply p={p} q={q} {n}^3 ({ndof} dofs)",
                   "mesh": [n, n, n], "p": p, "q": q, "parallelism": "host processes"},
        "cpu_baseline": {k: vals[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_ours(a):
    import torch

    from paper_2603_09038_b200 import Comm, PAOperator, build_mesh

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm(rank, world, local)
    p = a.p or 4
    q = a.q or p + 2
    n = a.n or (54 if p == 4 else SWEEP_N.get(p, 54))
    mesh = build_mesh(n, n, n * world)
    op = PAOperator(mesh, p, q, kind=a.kind, variant=a.variant, comm=comm)
    rng = np.random.default_rng(rank)
    x = torch.as_tensor(rng.standard_normal(op.num_dofs), device="cuda")
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    with sampler:
        for _ in range(max(3, a.warmup)):
            op.apply(x, out=y)
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(a.steps):
            op.apply(x, out=y)
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1) / a.steps
        # kernel-only timing for the roofline (events around the fused kernel,
        # on the operator's stream; median over the reps)
        reps = max(20, min(a.steps, 100))
        _, ms_kernel = op.time_apply(x, y, reps)
        # keep the same load until nvidia-smi has >= 3 samples (clock check only;
        # nothing here is timed)
        t_hold = time.time()
        while sampler.count() < 3 and time.time() - t_hold < 2.0:
            for _ in range(20):
                op.apply(x, out=y)
            torch.cuda.synchronize()
    ms = max_over_ranks(ms)
    ms_kernel = max_over_ranks(ms_kernel)
    ndof_global = op.num_global_dofs
    value = ndof_global / (ms * 1e-3) / 1e9

    # e2e: public API with host buffers (pinned), H2D + apply + D2H in the region
    xh = torch.empty(op.num_dofs, dtype=torch.float64, pin_memory=True)
    yh = torch.empty(op.num_dofs, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    xn, yn = xh.numpy(), yh.numpy()
    e2e_steps = max(3, min(a.steps, 50))
    for _ in range(2):
        op.apply_host(xn, yn)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        op.apply_host(xn, yn)
    barrier()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    e2e_value = ndof_global / (e2e_ms * 1e-3) / 1e9

    peak, peak_src = measured_peaks()
    alg_bytes = op.bytes_per_apply
    achieved = alg_bytes / (ms_kernel * 1e-3) / 1e9
    traffic = ncu_traffic(a.kind, p, n)
    clocks = sampler.summary()
    clocks["window"] = "nvidia-smi -lms 50 from warm-up start to the end of the kernel timing"
    sweep = None
    if a.sweep and rank == 0 and world == 1:
        sweep = run_sweep(a, peak)
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu_baseline:
            try:
                cpu = cpu_baseline(a.kind, n, p, q, a.cpu_seconds)
            except Exception as ex:  # reported, never fatal for the GPU number
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {ex}"}
        strat = "MF (matrix-free)" if op.variant == "mf" else "PA"
        work = (f"BP3 {strat} diffusion apply p={p} q={q}" if a.kind == "diffusion"
                else f"BP1 {strat} mass apply p={p} q={q}")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (x ~ N(0,1) seed=rank, unit-cube Cartesian hex mesh)",
            "config": {"workload": f"{work} {n}x{n}x{n * world} ({ndof_global} dofs)",
                       "mesh": [n, n, n * world], "p": p, "q": q,
                       "elements_per_gpu": n ** 3, "dofs_per_gpu": op.num_dofs,
                       "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                       "variant": op.variant,
                       "l2": ((f"inputs larger than L2 ({op.bytes_per_apply / 1e9:.2f} GB moved "
                               "per apply, no flush needed)") if op.bytes_per_apply > 126e6 else
                              "small config: L2-resident between steps (not a bandwidth number)"),
                       "launch": {"elems_per_block": op.info.elems_per_block,
                                  "threads": op.info.threads_per_block, "blocks": op.info.blocks}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src, "kernel_ms": ms_kernel,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel": f"fused apply kernel, variant {op.variant} (pa_pipe_kernel: gather, B/G, D, "
                                   "B^T/G^T, scatter-add in one launch)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * op.num_dofs,
                    "d2h_bytes_per_step": 8 * op.num_dofs, "ms_per_step": e2e_ms,
                    "path": "PAOperator.apply_host -> fk_op_apply_host (pinned host buffers)"},
            "gpu_launches": a.steps * (1 + (2 if world > 1 else 0)),
            "clocks": clocks,
        }
        if sweep is not None:
            line["sweep_file"] = a.sweep
        print(json.dumps(line), flush=True)
    op.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def run_cg(a):
    """BASELINE configs[3]/[4]: 100-iteration Jacobi-PCG, homogeneous Dirichlet on
    all faces, b ~ N(0,1) (seed = rank) with boundary entries zeroed, x0 = 0.
    weak: p=4, 92^3 elements per GPU (z-slabs of a 92x92x(92N) box);
    strong: p=6, fixed 98x98x96 box split into z-slabs.
    Metric: GDOF/s = global dofs x iterations / solve time (MFEM BP convention);
    the solve time includes the Jacobi-diagonal assembly (MAX over ranks)."""
    import torch

    from paper_2603_09038_b200 import Comm, PAOperator, build_mesh, cg_solve

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm(rank, world, local)
    if a.cg == "weak":
        p, n = a.p or 4, a.n or 92
        mesh, scaling = build_mesh(n, n, n * world), "weak"
    else:
        p, scaling = a.p or 6, "strong"
        mesh = build_mesh(98, 98, 96) if a.n is None else build_mesh(a.n, a.n, a.n)
    op = PAOperator(mesh, p, kind="diffusion", dirichlet=True, variant=a.variant, comm=comm)
    b = torch.as_tensor(np.random.default_rng(rank).standard_normal(op.num_dofs), device="cuda")
    op.set_essential(b, 0.0)
    iters = 100
    for _ in range(max(1, a.warmup // 3)):
        cg_solve(op, b, iters=5)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    x, hist = cg_solve(op, b, iters=iters)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        ndof = op.num_global_dofs
        print(json.dumps({
            "metric": f"GDOF/s of BP3 Jacobi-PCG ({scaling} scaling, {iters} iterations)",
            "value": ndof * iters / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "ms_per_iteration": ms / iters, "ms_solve": ms, "iterations": len(hist) - 1,
            "residual_0": float(hist[0]), "residual_final": float(hist[-1]),
            "higher_is_better": True, "scaling": scaling, "dtype": "f64",
            "config": {"workload": f"BP3 p={p} CG on {mesh.nx}x{mesh.ny}x{mesh.nz} ({ndof} dofs)",
                       "p": p, "variant": op.variant, "dofs_per_gpu": op.num_dofs},
        }), flush=True)
    op.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def run_mixed(a):
    """FusedPA apply of the acoustic-gravity block operator on 1 GPU at the
    paper's Table VII configuration (H1 p=4 / L2 p=3, q=5, 128^3 elements =
    537.7 M dofs; PAPER.md:647-664 reports 46.60 GDOF/s for DMMA Fused PA on
    GB200).  Inputs resident in HBM (dmat 18.9 GB > L2); GDOF/s = state dofs /
    apply time.  Also times one device RK4 step (4 applies + axpys)."""
    import torch

    from paper_2603_09038_b200 import MixedOperator, MixedState, build_mesh

    torch.cuda.set_device(0)
    p = a.p or 4
    n = a.n or 128
    strategy = "FusedMF" if a.variant == "mf" else "FusedPA"
    op = MixedOperator(build_mesh(n, n, n), p, p - 1, p + 1, strategy=strategy)
    g = torch.Generator(device="cuda").manual_seed(0)
    s = MixedState(torch.randn(op.u_shape, dtype=torch.float64, device="cuda", generator=g),
                   torch.randn(op.num_p, dtype=torch.float64, device="cuda", generator=g))
    out = op.zero_state(device=True)
    sampler = ClockSampler(0)
    with sampler:
        for _ in range(max(3, a.warmup)):
            op.apply(s, out=out)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(a.steps):
            op.apply(s, out=out)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / a.steps
        _, ms_kernel = op.time_apply(s, out, min(a.steps, 50))
        op.rk4(s, 1e-6, 1)
        torch.cuda.synchronize()
        ev0.record()
        op.rk4(s, 1e-6, 8)  # 8 steps per call: the state copy-in/out and finite check amortise
        ev1.record()
        torch.cuda.synchronize()
        ms_rk4 = ev0.elapsed_time(ev1) / 8
    peak, peak_src = measured_peaks()
    alg = op.bytes_per_apply
    published = 46.60 if strategy == "FusedPA" else 37.26  # PAPER.md:663 DMMA Fused PA / MF
    value = op.num_dofs / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": f"GDOF/s of the {strategy} acoustic-gravity block apply (H1 p=4 x L2 p=3, q=5)",
        "value": value, "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        f"vs_published_gb200_dmma_{strategy.lower()}": value / published, "dtype": "f64",
        "data": "synthetic (u, p ~ N(0,1)), unit-cube Cartesian hex mesh",
        "config": {"workload": f"BlockOperator {strategy} apply {n}^3 elements, order_p={p}, "
                               f"order_u={p - 1}, q={p + 1} ({op.num_dofs} dofs: "
                               f"{op.num_dofs - op.num_p} velocity + {op.num_p} pressure)",
                   "launch": {"elems_per_block": op.launch[0], "threads": op.launch[1],
                              "blocks": op.launch[2]},
                   "l2": "inputs larger than L2 (dmat 9 comps/point, ~19 GB)"},
        "roofline": {"bound": "hbm", "achieved": alg / (ms_kernel * 1e-3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": alg / (ms_kernel * 1e-3) / 1e9 / peak,
                     "peak_source": peak_src, "kernel_ms": ms_kernel,
                     "algorithmic_bytes_per_launch": alg},
        "rk4_step_ms": ms_rk4, "rk4_gdofs_per_apply": 4 * op.num_dofs / (ms_rk4 * 1e-3) / 1e9,
        "clocks": sampler.summary(),
    }), flush=True)
    op.close()


def run_sweep(a, peak):
    """p=1..8 BP3/BP1 sweep, DFMA vs DMMA, written as JSON lines to a file."""
    import torch

    from paper_2603_09038_b200 import PAOperator, build_mesh

    out = []
    cfgs = ([("dfma", c) for c in range(7)] + [("dmma", c) for c in range(3)]
            + [("eo", c) for c in range(36)] + [("mf", c) for c in range(11)])
    if a.sweep_cfgs:
        want = set(a.sweep_cfgs.split(","))
        cfgs = [vc for vc in cfgs if f"{vc[0]}{vc[1]}" in want]
    for kind in a.sweep_kinds.split(","):
        for p in [int(v) for v in a.sweep_orders.split(",")]:
            n = SWEEP_N[p]
            op = PAOperator(build_mesh(n, n, n), p, kind=kind)
            x = torch.randn(op.num_dofs, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            for variant, cfg in cfgs:
                try:
                    op.set_config(variant, cfg)
                except NotImplementedError:
                    continue
                op.time_apply(x, y, 5)
                ms_a, ms_k = op.time_apply(x, y, 30)
                rec = {"kind": kind, "p": p, "n": n, "variant": variant, "cfg": cfg, "ndof": op.num_dofs,
                       "ms_apply": ms_a, "ms_kernel": ms_k,
                       "gdofs": op.num_dofs / (ms_a * 1e-3) / 1e9,
                       "hbm_frac": op.bytes_per_apply / (ms_k * 1e-3) / 1e9 / peak,
                       "tflops": op.flops_per_apply / (ms_k * 1e-3) / 1e12,
                       "launch": [op.info.elems_per_block, op.info.threads_per_block, op.info.blocks]}
                out.append(rec)
                print(json.dumps(rec), file=sys.stderr, flush=True)
            op.close()
            del x, y
            torch.cuda.empty_cache()
    with open(a.sweep, "w") as f:
        for r in out:
            f.write(json.dumps(r) + "\n")
    return out


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.cg:
        run_cg(a)
    elif a.mixed:
        run_mixed(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
