"""Search shared-memory line layouts of the DFMA line kernel for minimum
wavefronts (design-time aid; see tools/smem_model.py for the bank model).

Each intermediate buffer (T1, T2, W, R) is a set of lines indexed by two 1D
indices; we choose its line numbering order, pitch and a per-line rotation of
the offsets, and each stage chooses the order in which lanes walk its lines.
The cost of a buffer depends only on (writer order, reader order, layout), so
the optimum is a small dynamic program over the five stage orders.

    python tools/smem_layout_search.py D Q NC E T
"""

from __future__ import annotations

import itertools
import sys
from functools import lru_cache

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from smem_model import wavefronts  # noqa: E402


def lanes_lines(n_lines_elem, E, T, order, n1, n2):
    """Per warp instruction group: list of 32 (e, i1, i2) or None.
    Stage line l (per element) -> (i1, i2): order 0: i1 = l % n1 ; order 1: i2 fastest."""
    out = []
    n = E * n_lines_elem
    for w0 in range(0, T, 32):
        lanes = []
        for l in range(32):
            t = w0 + l
            if t >= min(T, n):
                lanes.append(None)
                continue
            e, ll = divmod(t, n_lines_elem)
            if order == 0:
                lanes.append((e, ll % n1, ll // n1))
            else:
                lanes.append((e, ll // n2, ll % n2))
        if any(x is not None for x in lanes):
            out.append(lanes)
    return out


def addr(buf, e, s, i1, i2, off):
    n1, n2, ns, order, pitch, rot, est = buf
    line = i1 + n1 * i2 if order == 0 else i2 + n2 * i1
    return e * est + s * (n1 * n2 * pitch) + line * pitch + (off + rot * line) % pitch


def cost_buffer(buf, writer, reader):
    """writer/reader: (lanes, fn(lane_tuple, idx) -> (s, i1, i2, off), n_idx)."""
    tot = 0
    for lanes_groups, fn, nidx in (writer, reader):
        for lanes in lanes_groups:
            for idx in range(nidx):
                a = []
                for ln in lanes:
                    if ln is None:
                        a.append(None)
                    else:
                        s, i1, i2, off = fn(ln, idx)
                        a.append(addr(buf, ln[0], s, i1, i2, off))
                tot += wavefronts(a)
    return tot


def search(D, Q, NC, E, T):
    NA = 2 if NC == 3 else 1
    NR = 2 if NC == 3 else 1
    # stage line index spaces: A (j,k) D x D ; B (k,a) D x Q ; C (a,b) Q x Q ; D (a,k) Q x D ; E (j,k) D x D
    st = {"A": (D, D), "B": (D, Q), "C": (Q, Q), "D": (Q, D), "E": (D, D)}
    lanes = {(k, o): lanes_lines(v[0] * v[1], E, T, o, v[0], v[1]) for k, v in st.items() for o in (0, 1)}
    pitches = {"D": range(D, D + 9), "Q": range(Q, Q + 9)}

    def bufspec(n1, n2, ns, order, pitch, rot):
        return (n1, n2, ns, order, pitch, rot, (n1 * n2 * ns * pitch) | 1)

    # buffers: (line dims, offsets, ns, writer stage, reader stage, accessor fns)
    # T1: lines (k,a) offset j; writer A lane (j,k) -> for (s,a): (s,k,a,j); reader B lane (k,a) -> (s,k,a,j)
    defs = {
        "T1": ((D, Q), "D", NA, "A", "B",
               lambda ln, idx: (idx // Q, ln[2], idx % Q, ln[1]), NA * Q,
               lambda ln, idx: (idx // D, ln[1], ln[2], idx % D), NA * D),
        # T2: lines (a,b) offset k; writer B lane (k,a): (s, a, b, k); reader C lane (a,b): (s,a,b,k)
        "T2": ((Q, Q), "D", NC, "B", "C",
               lambda ln, idx: (idx // Q, ln[2], idx % Q, ln[1]), NC * Q,
               lambda ln, idx: (idx // D, ln[1], ln[2], idx % D), NC * D),
        # W: lines (a,k) offset b; writer C lane (a,b): (s,a,k,b); reader D lane (a,k): (s,a,k,b)
        "W": ((Q, D), "Q", NC, "C", "D",
              lambda ln, idx: (idx // D, ln[1], idx % D, ln[2]), NC * D,
              lambda ln, idx: (idx // Q, ln[1], ln[2], idx % Q), NC * Q),
        # R: lines (j,k) offset a; writer D lane (a,k): (s,j,k,a); reader E lane (j,k): (s,j,k,a)
        "R": ((D, D), "Q", NR, "D", "E",
              lambda ln, idx: (idx // D, idx % D, ln[2], ln[1]), NR * D,
              lambda ln, idx: (idx // Q, ln[1], ln[2], idx % Q), NR * Q),
    }

    @lru_cache(maxsize=None)
    def best_buffer(name, ow, orr):
        (n1, n2), pk, ns, ws, rs, wfn, wn, rfn, rn = defs[name]
        best = None
        for order, pitch, rot in itertools.product((0, 1), pitches[pk], (0, 1)):
            b = bufspec(n1, n2, ns, order, pitch, rot)
            c = cost_buffer(b, (lanes[(ws, ow)], wfn, wn), (lanes[(rs, orr)], rfn, rn))
            key = (c, pitch)
            if best is None or key < best[0]:
                best = (key, (order, pitch, rot))
        return best[0][0], best[1]

    # X read by A (lane (j,k) reads line (j,k) offset i), pitch choice, X written by cp.async (ignored)
    @lru_cache(maxsize=None)
    def best_x(oa):
        best = None
        for order, pitch, rot in itertools.product((0, 1), pitches["D"], (0, 1)):
            b = bufspec(D, D, 1, order, pitch, rot)
            c = cost_buffer(b, ([], None, 0), (lanes[("A", oa)], lambda ln, idx: (0, ln[1], ln[2], idx), D))
            if best is None or (c, pitch) < best[0]:
                best = ((c, pitch), (order, pitch, rot))
        return best[0][0], best[1]

    # D data read by C: layout chosen to match C's lane order -> consecutive lanes, consecutive words
    results = []
    for oa, ob, oc, od, oe in itertools.product((0, 1), repeat=5):
        tot = best_x(oa)[0] + best_buffer("T1", oa, ob)[0] + best_buffer("T2", ob, oc)[0] \
            + best_buffer("W", oc, od)[0] + best_buffer("R", od, oe)[0]
        results.append((tot, (oa, ob, oc, od, oe)))
    results.sort()
    base = best_x(0)[0] + best_buffer("T1", 0, 0)[0] + best_buffer("T2", 0, 0)[0] \
        + best_buffer("W", 0, 0)[0] + best_buffer("R", 0, 0)[0]
    return results, base, best_x, best_buffer


def main():
    D, Q, NC, E, T = (int(a) for a in sys.argv[1:6])
    results, base, best_x, best_buffer = search(D, Q, NC, E, T)
    print(f"orders all-0 (best pads/rot): {base / E:.1f} wf/elem")
    for tot, o in results[:4]:
        oa, ob, oc, od, oe = o
        print(f"orders {o}: {tot / E:.1f} wf/elem  X{best_x(oa)[1]} T1{best_buffer('T1', oa, ob)[1]} "
              f"T2{best_buffer('T2', ob, oc)[1]} W{best_buffer('W', oc, od)[1]} R{best_buffer('R', od, oe)[1]}")


if __name__ == "__main__":
    main()
