#!/usr/bin/env python
"""Benchmark: GDOF/s of the PA operator apply (BP3 diffusion) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--p 4] [--n 54] [--variant auto|dfma|dmma] [--sweep FILE]

A step is one operator apply y = A x (gather, B/G contractions, PA data D,
transposed contractions, scatter-add, and for N>1 the interface exchange)
over the whole mesh, inputs resident in HBM.  Default workload =
BASELINE.json configs[1]: BP3, p=4, q=6, 54^3 elements (10,218,313 dofs).
For N>1 every rank owns a 54^3-element z-slab of a 54x54x(54N) mesh (weak
scaling) and the slabs exchange their interface planes (peer-memory
transport over NVLink by default, ``--transport nccl`` for NCCL).  Without
torchrun, ``--gpus N`` launches its own N ranks (torch.distributed.run on
127.0.0.1).

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
CPU algorithm (the oracle/ restatement, per-element NumPy path exactly as
feklab executes it) over all host cores: every one of the K timed steps is a
bounded element sample of the same workload, so the K + W steps take a few
minutes at most.
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
    ap.add_argument("--n", "--elems", dest="n", type=int, default=None,
                    help="elements per direction (per-rank slab is n^3)")
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
    ap.add_argument("--deterministic", action="store_true",
                    help="verification mode: colour-ordered elements, bitwise reproducible applies")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="z-slab exchange for N>1: peer-memory mailboxes (default) or NCCL")
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


# measured FP64 throughput of this pool's B200 (tools/fp64_peak.cu,
# profiles/r01_fp64_peak.txt: DFMA 37.07, DMMA 37.16 TFLOP/s; they share the pipe)
FP64_TFLOPS = 37.07


def ncu_traffic(kind, p, n, variant, cfg):
    """DRAM bytes per launch of the fused kernel of exactly this launch
    geometry (variant + cfg) from the committed ncu summary, else None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(f"{kind}_p{p}_n{n}_{variant}{cfg}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


def workload_config(kind, p, q, n, world, mf=False):
    """The config dict BOTH arms print (ours and --impl reference)."""
    ndof = (n * p + 1) * (n * p + 1) * (n * world * p + 1)
    strat = "MF (matrix-free)" if mf else "PA"
    work = (f"BP3 {strat} diffusion apply p={p} q={q}" if kind == "diffusion"
            else f"BP1 {strat} mass apply p={p} q={q}")
    return {"workload": f"{work} {n}x{n}x{n * world} ({ndof} dofs)",
            "mesh": [n, n, n * world], "p": p, "q": q, "elements_per_gpu": n ** 3,
            "parallelism": f"z-slab x{world}" if world > 1 else "single GPU"}


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
    e0, e1 = args
    from oracle import bp

    P, x, n, nz = _CPU["problem"], _CPU["x"], _CPU["n"], _CPU["nz"]  # inherited via fork
    y = _CPU.get("y")
    if y is None:
        y = _CPU["y"] = np.zeros(P.ndof)
    t = time.perf_counter()
    ids = bp.gather_ids_elements(n, n, nz, P.d, e0, e1)
    xe = x[ids]                                     # Restriction.gather (mesh.py:130-131)
    ye = P.element_apply(xe, batched=False)         # per-element chains (tensor.py:220-283)
    np.add.at(y, ids.ravel(), ye.ravel())           # Restriction.scatter_add (mesh.py:133-137)
    return e1 - e0, time.perf_counter() - t


class CpuRef:
    """The reference's CPU path (oracle/bp.py per-element restatement of
    feklab, bit-identical to it) on the host cores: a persistent fork pool,
    each worker applying a contiguous element range of the n x n x nz mesh."""

    def __init__(self, kind, n, nz, p, q, cores=None):
        import multiprocessing as mp

        from oracle import bp

        self.cores = cores or os.cpu_count() or 1
        P = bp.Problem(kind, 2, 2, 2, p, q)
        # the element operator only depends on (p, q, h): take h of the n^3 mesh
        P.jd, P.detj = bp.jacobian(n, n, n)
        P.jinv = 1.0 / P.jd
        P.wdet = bp.quad_weights_3d(P.w) * P.detj
        P.ndof = bp.num_dofs(n, n, nz, P.d)
        _CPU.clear()
        _CPU.update(problem=P, x=np.random.default_rng(0).standard_normal(P.ndof), n=n, nz=nz)
        self.kind, self.n, self.nz, self.p, self.P = kind, n, nz, p, P
        self.nel, self.ndof = n * n * nz, P.ndof
        xe = np.random.default_rng(0).standard_normal((8, P.d ** 3))
        P.element_apply(xe, batched=False)
        t = time.perf_counter()
        P.element_apply(np.repeat(xe, 4, axis=0), batched=False)
        self.sec_per_el = (time.perf_counter() - t) / 32
        self.pool = mp.get_context("fork").Pool(self.cores)
        self.offset = 0

    def per_worker(self, seconds):
        return int(max(1, min(seconds / max(self.sec_per_el, 1e-7), self.nel // self.cores)))

    def step(self, per_worker):
        """One bounded sample: every worker applies per_worker elements.
        Returns (elements, wall seconds, slowest worker seconds)."""
        jobs = []
        for w in range(self.cores):
            e0 = (self.offset + w * per_worker) % max(1, self.nel - per_worker)
            jobs.append((e0, e0 + per_worker))
        self.offset = (self.offset + self.cores * per_worker) % max(1, self.nel)
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, jobs)
        wall = time.perf_counter() - t0
        return sum(r[0] for r in res), wall, max(r[1] for r in res)

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_baseline(kind, n, p, q, seconds, cores=None, nz=None):
    """GDOF/s of the reference's CPU path on a bounded sample (~``seconds``
    per worker), extrapolated by the sample's share of the elements."""
    ref = CpuRef(kind, n, nz or n, p, q, cores)
    try:
        pw = ref.per_worker(seconds / 2)
        best = None
        for _ in range(2):
            el, wall, slow = ref.step(pw)
            best = slow if best is None else min(best, slow)
        dofs = ref.ndof * el / ref.nel
        return {"value": dofs / best / 1e9, "unit": UNIT, "cores": ref.cores, "kind": "port",
                "cpu_model": cpu_model(),
                "sample": f"{el} of {ref.nel} elements ({kind} p={p} {n}x{n}x{nz or n}), per-element "
                          f"NumPy restatement of feklab's path, {ref.cores} processes, best of 2, "
                          f"throughput scaled by element share"}
    finally:
        ref.close()


def run_reference(a):
    """The reference arm: the reference's CPU algorithm on this box's host
    cores, on our arm's workload/config/metric.  Exactly ``steps`` timed
    steps after ``warmup`` untimed ones; each step is one bounded element
    sample (all cores), sized so the whole run takes ~2 minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = a.gpus
    p = a.p or 4
    q = a.q or p + 2
    n = a.n or (54 if p == 4 else SWEEP_N.get(p, 54))
    ref = CpuRef(a.kind, n, n * world, p, q)
    budget = min(5.0, max(0.05, 120.0 / max(1, a.steps + a.warmup)))  # seconds per step
    pw = ref.per_worker(0.8 * budget)
    for _ in range(a.warmup):
        ref.step(pw)
    t0 = time.perf_counter()
    els = 0
    for _ in range(a.steps):
        el, _, _ = ref.step(pw)
        els += el
    wall = time.perf_counter() - t0
    ref.close()
    dofs = ref.ndof * els / ref.nel
    v = dofs / wall / 1e9
    sample = (f"{els // max(1, a.steps)} of {ref.nel} elements per step ({ref.cores} processes x {pw}), "
              f"per-element NumPy restatement of feklab's path (oracle/bp.py), GDOF/s = "
              f"element share x {ref.ndof} dofs / wall time of the {a.steps} timed steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": wall * 1e3 / max(1, a.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (x ~ N(0,1), seed 0)",
        "config": workload_config(a.kind, p, q, n, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": ref.cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def init_ranks(a):
    """(world, rank, local, dist|None, comm|None): torch.distributed over NCCL
    for the bootstrap and the max-over-ranks timing, the library's own
    communicator (``--transport``) for the exchange."""
    import torch

    from paper_2603_09038_b200 import Comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # FK_BENCH_DEVICE=d: every rank on device d (exercises the multi-rank code
    # path on a one-GPU box; processes then time-slice the GPU, so the number
    # is not a scaling measurement) with a gloo bootstrap
    shared = os.environ.get("FK_BENCH_DEVICE")
    if shared is not None:
        local = int(shared)
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"--gpus {a.gpus}: rank {rank} needs cuda:{local} but {torch.cuda.device_count()} "
                         f"GPU(s) are visible (one process per GPU; FK_BENCH_DEVICE=0 runs every rank on "
                         f"cuda:0 to exercise the multi-rank path, not to measure scaling)")
    torch.cuda.set_device(local)
    if world == 1:
        return world, rank, local, None, None
    import torch.distributed as dist

    # NCCL's init log (ranks, devices, NVLink/NVLS topology) to stderr, so the
    # rank count can be checked while stdout keeps its single JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if shared is not None:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = Comm(rank, world, local, transport=a.transport)
    print(f"[fk] rank {rank}/{world} on cuda:{local} ({torch.cuda.get_device_name(local)}), "
          f"z-slab exchange over {a.transport}", file=sys.stderr, flush=True)
    return world, rank, local, dist, comm


def trace(msg):
    """Per-rank phase log on stderr for multi-rank runs (FK_BENCH_TRACE=1)."""
    if os.environ.get("FK_BENCH_TRACE"):
        print(f"[fk {time.strftime('%H:%M:%S')} rank {os.environ.get('RANK', '0')}] {msg}",
              file=sys.stderr, flush=True)


def run_ours(a):
    import torch

    from paper_2603_09038_b200 import PAOperator, build_mesh

    world, rank, local, dist, comm = init_ranks(a)
    p = a.p or 4
    q = a.q or p + 2
    n = a.n or (54 if p == 4 else SWEEP_N.get(p, 54))
    mesh = build_mesh(n, n, n * world)
    op = PAOperator(mesh, p, q, kind=a.kind, variant=a.variant, comm=comm,
                    deterministic=a.deterministic)
    if comm is not None:
        print(f"[fk] rank {rank}: exchange transport in use: {comm.transport}", file=sys.stderr, flush=True)
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

    def timed_applies(o, steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            o.apply(x, out=y)
        ev1.record(stream)
        barrier()
        return ev0.elapsed_time(ev1) / steps

    single_ms = None
    if world > 1:
        # weak-scaling reference: the same per-rank slab alone on this GPU (no
        # exchange), timed the same way, before the multi-rank run
        trace("solo slab")
        solo = PAOperator(build_mesh(n, n, n), p, q, kind=a.kind, variant=a.variant,
                          deterministic=a.deterministic)
        for _ in range(max(3, a.warmup)):
            solo.apply(x, out=y)
        barrier()
        single_ms = max_over_ranks(timed_applies(solo, a.steps))
        solo.close()
    trace("warm-up")
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(max(3, a.warmup)):
            op.apply(x, out=y)
        barrier()
        trace("timed applies")
        ms = timed_applies(op, a.steps)
        trace("kernel timing")
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

    trace("e2e")
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
    mf = op.variant == "mf"
    alg_bytes = op.bytes_per_apply
    if mf:
        # matrix-free: no PA data stream; bound by the FP64 pipe (and shared
        # memory), so rate the kernel against the measured FP64 peak
        achieved = op.flops_per_apply / (ms_kernel * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": FP64_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_TFLOPS, "peak_source": "measured (profiles/r01_fp64_peak.txt)",
                "algorithmic_flops_per_launch": op.flops_per_apply,
                "hbm_achieved_gbs": alg_bytes / (ms_kernel * 1e-3) / 1e9}
    else:
        achieved = alg_bytes / (ms_kernel * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes}
    roof["traffic"] = ncu_traffic(a.kind, p, n, op.variant, op.info.cfg)
    roof["kernel_ms"] = ms_kernel
    roof["kernel"] = (f"fused apply kernel, variant {op.variant} cfg {op.info.cfg} (pa_pipe_kernel: "
                      "gather, B/G, D, B^T/G^T, scatter-add in one launch)")
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
        # kernels of ours per apply: the fused kernel (3 launches: two boundary
        # layers + interior, when a multi-rank slab has >= 3 layers) and the
        # four exchange kernels (credit wait, put, arrival wait, add)
        per_apply = 1 if world == 1 else ((3 if n >= 3 else 1) + (4 if comm.transport == "p2p" else 2))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (x ~ N(0,1) seed=rank, unit-cube Cartesian hex mesh)",
            "config": workload_config(a.kind, p, q, n, world),
            "impl_config": {
                "variant": op.variant, "cfg": op.info.cfg, "dofs_per_gpu": op.num_dofs,
                "transport": comm.transport if comm is not None else None,
                "deterministic": a.deterministic,
                "l2": ((f"inputs larger than L2 ({op.bytes_per_apply / 1e9:.2f} GB moved "
                        "per apply, no flush needed)") if op.bytes_per_apply > 126e6 else
                       "small config: L2-resident between steps (not a bandwidth number)"),
                "launch": {"elems_per_block": op.info.elems_per_block,
                           "threads": op.info.threads_per_block, "blocks": op.info.blocks}},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * op.num_dofs,
                    "d2h_bytes_per_step": 8 * op.num_dofs, "ms_per_step": e2e_ms,
                    "path": "PAOperator.apply_host -> fk_op_apply_host (pinned host buffers)"},
            "gpu_launches": a.steps * per_apply,
            "clocks": clocks,
        }
        if single_ms is not None:
            line["weak_scaling"] = {"single_gpu_ms_per_apply": single_ms, "ms_per_apply": ms,
                                    "efficiency": single_ms / ms,
                                    "note": "same per-rank slab alone on each GPU (no exchange), max over ranks"}
        if sweep is not None:
            line["sweep_file"] = a.sweep
        print(json.dumps(line), flush=True)
    op.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def cpu_cg_baseline(n, nz, p, seconds):
    """The oracle PCG loop (oracle/bp.py Problem.pcg, the reference's path for
    the apply) per iteration on the host cores: apply throughput from a
    bounded element sample of the CG mesh (CpuRef, all cores) plus the
    loop's vector work (x, r, z, p updates and the two dots, NumPy) timed on
    a slice and scaled to the full vectors."""
    ref = CpuRef("diffusion", n, nz, p, p + 2)
    try:
        pw = ref.per_worker(seconds / 2)
        best = None
        for _ in range(2):
            el, _, slow = ref.step(pw)
            best = slow if best is None else min(best, slow)
        t_apply = best * ref.nel / el
    finally:
        ref.close()
    m = min(ref.ndof, 4_000_000)
    rng = np.random.default_rng(0)
    xv, r, pv, Ap, dinv = (rng.standard_normal(m) for _ in range(5))
    t = time.perf_counter()
    for _ in range(3):
        den = float(pv @ Ap)
        alpha = 1.0 / (1.0 + abs(den))
        xv += alpha * pv
        r -= alpha * Ap
        z = dinv * r
        bn = float(r @ z)
        pv = z + (bn / (1.0 + bn)) * pv
    t_vec = (time.perf_counter() - t) / 3 * ref.ndof / m
    t_iter = t_apply + t_vec
    return {"value": ref.ndof / t_iter / 1e9, "unit": UNIT, "cores": ref.cores, "kind": "port",
            "cpu_model": cpu_model(), "s_per_iteration": t_iter,
            "sample": f"oracle PCG iteration = apply ({el} of {ref.nel} elements on {ref.cores} processes, "
                      f"scaled by element share: {t_apply:.2f} s) + vector updates/dots (NumPy, 1 thread, "
                      f"{m} of {ref.ndof} entries, scaled: {t_vec:.2f} s)"}


def run_cg(a):
    """BASELINE configs[3]/[4]: 100-iteration Jacobi-PCG, homogeneous Dirichlet on
    all faces, b ~ N(0,1) (seed = rank) with boundary entries zeroed, x0 = 0.
    weak: p=4, 92^3 elements per GPU (z-slabs of a 92x92x(92N) box);
    strong: p=6, fixed 98x98x96 box split into z-slabs.
    Metric: GDOF/s = global dofs x iterations / solve time (MFEM BP convention);
    the solve time includes the Jacobi-diagonal assembly (MAX over ranks).
    For N > 1 the same solve is first timed on one GPU (weak: the per-rank
    slab on every GPU; strong: the whole box on rank 0) for the efficiency."""
    import torch

    from paper_2603_09038_b200 import PAOperator, build_mesh, cg_solve

    world, rank, local, dist, comm = init_ranks(a)
    if a.cg == "weak":
        p, n = a.p or 4, a.n or 92
        dims, scaling = (n, n, n * world), "weak"
    else:
        p, scaling = a.p or 6, "strong"
        dims = (98, 98, 96) if a.n is None else (a.n, a.n, a.n)
    iters = 100

    def solve_ms(op, b):
        for _ in range(max(1, a.warmup // 3)):
            cg_solve(op, b, iters=5)
        torch.cuda.synchronize()
        if op.comm is not None:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        _, hist = cg_solve(op, b, iters=iters)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), hist

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    single_ms = None
    if world > 1 and (scaling == "weak" or rank == 0):
        solo_dims = (dims[0], dims[1], dims[2] // world) if scaling == "weak" else dims
        solo = PAOperator(build_mesh(*solo_dims), p, kind="diffusion", dirichlet=True, variant=a.variant,
                          deterministic=a.deterministic)
        bs = torch.as_tensor(np.random.default_rng(rank).standard_normal(solo.num_dofs), device="cuda")
        solo.set_essential(bs, 0.0)
        single_ms, _ = solve_ms(solo, bs)
        solo.close()
        del bs
        torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
        single_ms = max_over_ranks(single_ms or 0.0)
    op = PAOperator(build_mesh(*dims), p, kind="diffusion", dirichlet=True, variant=a.variant, comm=comm,
                    deterministic=a.deterministic)
    b = torch.as_tensor(np.random.default_rng(rank).standard_normal(op.num_dofs), device="cuda")
    op.set_essential(b, 0.0)
    sampler = ClockSampler(local)
    with sampler:
        ms, hist = solve_ms(op, b)
    ms = max_over_ranks(ms)
    if rank == 0:
        ndof = op.num_global_dofs
        cpu = None
        if not a.no_cpu_baseline:
            try:
                cpu = cpu_cg_baseline(dims[0], dims[2], p, a.cpu_seconds)
            except Exception as ex:
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {ex}"}
        line = {
            "metric": f"GDOF/s of BP3 Jacobi-PCG ({scaling} scaling, {iters} iterations)",
            "value": ndof * iters / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "ms_per_iteration": ms / iters, "ms_solve": ms, "iterations": len(hist) - 1,
            "residual_0": float(hist[0]), "residual_final": float(hist[-1]),
            "higher_is_better": True, "scaling": scaling, "dtype": "f64",
            "data": "synthetic (b ~ N(0,1) seed=rank, boundary zeroed; x0 = 0)",
            "config": {"workload": f"BP3 p={p} CG on {dims[0]}x{dims[1]}x{dims[2]} ({ndof} dofs)",
                       "mesh": list(dims), "p": p, "q": p + 2, "iterations": iters,
                       "parallelism": f"z-slab x{world}" if world > 1 else "single GPU"},
            "impl_config": {"variant": op.variant, "cfg": op.info.cfg, "dofs_per_gpu": op.num_dofs,
                            "transport": comm.transport if comm is not None else None,
                            "deterministic": a.deterministic},
            "cpu_baseline": cpu,
            "clocks": sampler.summary(),
        }
        if single_ms:
            eff = single_ms / ms if scaling == "weak" else single_ms / (world * ms)
            line[f"{scaling}_scaling"] = {"single_gpu_ms_solve": single_ms, "ms_solve": ms,
                                          "efficiency": eff}
        print(json.dumps(line), flush=True)
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
    cfgs = ([("dfma", c) for c in range(7)] + [("dmma", c) for c in range(15)]
            + [("eo", c) for c in range(62)] + [("mf", c) for c in range(11)])
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


def spawn_ranks(a) -> int:
    """--gpus N without torchrun: launch N ranks of this script on 127.0.0.1."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    # torchrun's own parser would take "--n" as an abbreviation of its options
    cmd += ["--elems" + v[3:] if v == "--n" or v.startswith("--n=") else v for v in sys.argv[1:]]
    print(f"[fk] spawning {a.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(spawn_ranks(a))
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
