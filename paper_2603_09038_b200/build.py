"""Build libfk_b200.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2603_09038_b200.build [--force] [-j N]

Each order's fused kernels are one translation unit (pa_inst.cu with
-DFK_P=p), compiled in parallel, then linked with the C-ABI (fk_api.cu) and
the NCCL plumbing (fk_comm.cu).  The .so lands next to this file, so it
travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libfk_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
ORDERS = range(1, 9)


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def nccl_include() -> list[str]:
    try:
        import nvidia.nccl  # type: ignore

        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc]
    except Exception:
        pass
    if os.path.exists("/usr/include/nccl.h"):
        return []
    raise RuntimeError("nccl.h not found (pip nvidia-nccl or /usr/include)")


def flags() -> list[str]:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                   "-Xptxas", "-warn-spills", ] + nccl_include()


def sources():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "fk.h"))
    units = [(f"pa_p{p}", "pa_inst.cu", [f"-DFK_P={p}"]) for p in ORDERS]
    units += [(f"mix_p{p}", "mix_inst.cu", [f"-DFK_MIX_P={p}"]) for p in range(2, 9)]
    units += [("fk_api", "fk_api.cu", []), ("fk_comm", "fk_comm.cu", []), ("fk_mixed", "fk_mixed.cu", [])]
    return units, deps


def _compile(unit):
    name, src, extra = unit
    out = os.path.join(OBJ, name + ".o")
    cmd = [nvcc()] + flags() + extra + ["-c", os.path.join(CSRC, src), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    units, deps = sources()
    newest = max(os.path.getmtime(d) for d in deps + [os.path.abspath(__file__)])
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = jobs or min(len(units), os.cpu_count() or 4)
    objs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for out, err in ex.map(_compile, units):
            objs.append(out)
            if verbose and err.strip():
                sys.stderr.write(err)
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args(argv)
    print(build(a.force, a.j, a.v))


if __name__ == "__main__":
    main()
