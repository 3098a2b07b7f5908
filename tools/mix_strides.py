"""Shared-memory stride search for the acoustic-gravity kernel (mix_pipe.cuh).

Each intermediate buffer's two access patterns (writer stage, reader stage,
fixed thread->line maps of mix_pipe.cuh; the pressure and velocity line
groups are warp-aligned, so they never share an instruction) are scored
with the half-warp bank model of tools/smem_strides.py over every nesting
order and padding of the buffer's strides.  For the velocity buffers the
component r is a lane index (3 r-blocks of lines), so its stride is searched
too.  Prints a MixStrides<DP, DU, Q> specialisation for mix_pipe.cuh.

    python tools/mix_strides.py DP DU Q [E]
"""

from __future__ import annotations

import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from smem_strides import cost_many  # noqa: E402


def instrs(n_lines, lane_fn, loops, E=1):
    """Warp-aligned group of E*n_lines lines; lane l -> (comp_lane, i1, i2, i3) for loop vals."""
    I, M = [], []
    tot = E * n_lines
    for w0 in range(0, tot, 32):
        for lv in itertools.product(*[range(n) for n in loops]):
            idx = np.zeros((32, 4), np.int64)
            msk = np.zeros(32, bool)
            for l in range(32):
                t = w0 + l
                if t >= tot:
                    continue
                e, ll = divmod(t, n_lines)
                c, i1, i2, i3 = lane_fn(ll, *lv)
                idx[l] = (c + 3 * e, i1, i2, i3)  # elements after the 3 r-blocks
                msk[l] = True
            I.append(idx)
            M.append(msk)
    return np.array(I), np.array(M)


def layouts(n, ncl):
    """(strides (cs, s1, s2, s3), comp size) candidates; ncl = lane-level components."""
    out = []
    for perm in itertools.permutations(range(3)):
        ni, nm, no = (n[p] for p in perm)
        for p1, p2 in itertools.product(range(16), range(16)):
            sm = ni + p1
            so = sm * (nm - 1) + ni + p2
            size = so * (no - 1) + sm * (nm - 1) + ni
            st = [0, 0, 0]
            st[perm[0]], st[perm[1]], st[perm[2]] = 1, sm, so
            for p3 in (range(16) if ncl > 1 else [0]):
                out.append(((size + p3, *st), size))
    return out


def search(DP, DU, Q, E=1):
    bufs = {
        # name: (extents (i1,i2,i3), lane comps, writer (n, fn, loops), reader (n, fn, loops))
        "T1P": ((Q, DP, DP), 1,
                (DP * DP, lambda l, s, a: (0, a, l % DP, l // DP), [2, Q]),
                (Q * DP, lambda l, s, j: (0, l // DP, j, l % DP), [2, DP])),
        "T1U": ((Q, DU, DU), 3,
                (3 * DU * DU, lambda l, a: (l // (DU * DU), a, (l % (DU * DU)) % DU, (l % (DU * DU)) // DU), [Q]),
                (3 * Q * DU, lambda l, j: (l // (Q * DU), (l % (Q * DU)) // DU, j, (l % (Q * DU)) % DU), [DU])),
        "T2P": ((Q, Q, DP), 1,
                (Q * DP, lambda l, s, b: (0, l // DP, b, l % DP), [3, Q]),
                (Q * Q, lambda l, s, k: (0, l % Q, l // Q, k), [3, DP])),
        "T2U": ((Q, Q, DU), 3,
                (3 * Q * DU, lambda l, b: (l // (Q * DU), (l % (Q * DU)) // DU, b, (l % (Q * DU)) % DU), [Q]),
                (Q * Q, lambda l, r, k: (r, l % Q, l // Q, k), [3, DU])),
        "WU": ((Q, Q, DU), 3,
               (Q * Q, lambda l, r, k: (r, l % Q, l // Q, k), [3, DU]),
               (3 * Q * DU, lambda l, b: (l // (Q * DU), (l % (Q * DU)) % Q, b, (l % (Q * DU)) // Q), [Q])),
        "WP": ((Q, Q, DP), 1,
               (Q * Q, lambda l, s, k: (0, l % Q, l // Q, k), [3, DP]),
               (Q * DP, lambda l, s, b: (0, l % Q, b, l // Q), [3, Q])),
        "RU": ((Q, DU, DU), 3,
               (3 * Q * DU, lambda l, j: (l // (Q * DU), (l % (Q * DU)) % Q, j, (l % (Q * DU)) // Q), [DU]),
               (3 * DU * DU, lambda l, a: (l // (DU * DU), a, (l % (DU * DU)) % DU, (l % (DU * DU)) // DU), [Q])),
        "RP": ((Q, DP, DP), 1,
               (Q * DP, lambda l, s, j: (0, l % Q, j, l // Q), [2, DP]),
               (DP * DP, lambda l, s, a: (0, a, l % DP, l // DP), [2, Q])),
    }
    out = {}
    for name, (ext, ncl, wr, rd) in bufs.items():
        Iw, Mw = instrs(wr[0], wr[1], wr[2], E)
        Ir, Mr = instrs(rd[0], rd[1], rd[2], E)
        cands = layouts(ext, ncl)
        lay = np.array([c[0] for c in cands], np.int64)
        c = cost_many(lay, Iw, Mw) + cost_many(lay, Ir, Mr)
        i = np.lexsort((np.array([cd[1] for cd in cands]), c))[0]
        # the current (default) layout of mix_pipe.cuh for comparison
        out[name] = (int(c[i]), tuple(int(v) for v in lay[i]), cands[i][1])
    return out


if __name__ == "__main__":
    DP, DU, Q = (int(a) for a in sys.argv[1:4])
    E = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    res = search(DP, DU, Q, E)
    tot = 0
    for k, (c, lay, size) in res.items():
        tot += c
        print(f"{k:4s} {c:5d} wf  (cs, s1, s2, s3) = {lay}  comp size {size}")
    print("total", tot)
