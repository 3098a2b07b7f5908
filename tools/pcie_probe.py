"""PCIe probe for the e2e path: pinned H2D / D2H alone and overlapped, and
PAOperator.apply_host at several z-chunk counts (FK_HOST_CHUNKS)."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def copies(nbytes):
    n = nbytes // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                if name in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        d.copy_(h, non_blocking=True)
                if name in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 10
        out[name] = {"ms": dt * 1e3, "GB/s": nbytes / dt / 1e9}
    return out


def main():
    from paper_2603_09038_b200 import PAOperator, build_mesh

    op = PAOperator(build_mesh(54, 54, 54), 4)
    nb = op.num_dofs * 8
    res = {"bytes": nb, "copies": copies(nb)}
    xh = torch.empty(op.num_dofs, dtype=torch.float64, pin_memory=True).numpy()
    yh = torch.empty(op.num_dofs, dtype=torch.float64, pin_memory=True).numpy()
    xh[:] = np.random.default_rng(0).standard_normal(op.num_dofs)
    for ramp in ("0", "1"):
        os.environ["FK_HOST_RAMP"] = ramp
        for k in (4, 8, 12, 15):
            os.environ["FK_HOST_CHUNKS"] = str(k)
            for _ in range(3):
                op.apply_host(xh, yh)
            t0 = time.perf_counter()
            for _ in range(30):
                op.apply_host(xh, yh)
            dt = (time.perf_counter() - t0) / 30
            res[f"apply_host_K{k}_ramp{ramp}"] = {"ms": dt * 1e3, "GDOF/s": op.num_dofs / dt / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
