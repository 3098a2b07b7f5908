"""Shared-memory layout search for the even-odd line kernel (design-time aid).

Generalises tools/smem_layout_search.py: every intermediate buffer of the
fused apply (X, T1, T2, W, R) gets an arbitrary padded linear layout

    word(e, s, i1, i2, i3) = e*se + s*ss + i1*s1 + i2*s2 + i3*s3

(any nesting order of the three spatial indices, any padding of the middle,
outer and element strides), and every stage an arbitrary thread->line map
(element-major or element-minor, either index fastest).  Cost = 128-byte
shared-memory wavefronts per element under the half-warp bank model of
tools/smem_model.py (an 8-byte access is served per half-warp; wavefronts =
max number of distinct words per 8-byte bank pair).  The per-buffer optimum
depends only on (writer map, reader map), so the stage maps are chosen by
exhaustive enumeration over the cached per-buffer optima.

Canonical index order of each buffer (pa_dfma_eo.cuh, FoldLayout):
    X  (i, j, k)     dof x, y, z          written by the gather, read by A
    T1 (a, j, k)     quad x, dof y, z     A -> B        (NA components)
    T2 (a, b, k)     quad x, y, dof z     B -> C        (NC components)
    W  (a, b, k)                          C -> D        (NC components)
    R  (a, j, k)                          D -> E        (NR components)
Stage line spaces: A (j,k)  B (a,k)  C (a,b)  D (a,k)  E (j,k).

    python tools/smem_strides.py D Q NC E T [--ip]
"""

from __future__ import annotations

import itertools
import sys

import numpy as np

MAPS = (0, 1, 2, 3)  # 0: e-major p1 fastest, 1: e-major p2 fastest, 2: e-minor p1 fastest, 3: e-minor p2


def thread_lines(m, E, T, n1, n2):
    """Per warp (over passes): array (32, 3) of (e, p1, p2) and mask."""
    L = n1 * n2
    n = E * L
    out = []
    for t0 in range(0, n, T):
        for w0 in range(0, T, 32):
            idx = np.zeros((32, 3), np.int64)
            msk = np.zeros(32, bool)
            for l in range(32):
                t = t0 + w0 + l
                if w0 + l >= T or t >= n:
                    continue
                if m in (0, 1):
                    e, ll = divmod(t, L)
                else:
                    ll, e = divmod(t, E)
                if m in (0, 2):
                    p2, p1 = divmod(ll, n1)
                else:
                    p1, p2 = divmod(ll, n2)
                idx[l] = (e, p1, p2)
                msk[l] = True
            if msk.any():
                out.append((idx, msk))
    return out


def instrs(warps, place, loops):
    """Expand per-warp lanes into instructions.  place(e,p1,p2,*loopvals) -> (e,i1,i2,i3)
    vectorised over lanes; loops = list of loop extents (component loop excluded)."""
    I, M = [], []
    for idx, msk in warps:
        for lv in itertools.product(*[range(n) for n in loops]):
            I.append(np.stack(place(idx[:, 0], idx[:, 1], idx[:, 2], *lv), axis=1))
            M.append(msk)
    return np.array(I), np.array(M)


def cost_many(lays, I, M):
    """lays (L,4) strides for (e,i1,i2,i3); I (n,32,4); M (n,32) -> (L,) wavefronts."""
    tot = np.zeros(len(lays), np.int64)
    n = I.shape[0]
    half = (np.arange(32) >= 16).astype(np.int64)
    for c0 in range(0, len(lays), 2048):
        lay = lays[c0:c0 + 2048]
        nl = len(lay)
        w = np.einsum("lk,nak->lna", lay, I) % 16  # bank pair of every lane
        # one bincount over (layout, instruction, half-warp, bank)
        key = ((np.arange(nl)[:, None, None] * n + np.arange(n)[None, :, None]) * 2 + half) * 16 + w
        cnt = np.bincount(key[:, M].ravel(), minlength=nl * n * 32).reshape(nl, n * 2, 16)
        tot[c0:c0 + 2048] += cnt.max(-1).sum(-1)
    return tot


def layouts(n):
    """All candidate strides (se, s1, s2, s3) and sizes for extents n = (n1, n2, n3)."""
    out = []
    for perm in itertools.permutations(range(3)):
        ni, nm, no = (n[p] for p in perm)
        for p1, p2, p3 in itertools.product(range(16), range(16), range(16)):
            si = 1
            sm = ni + p1
            so = sm * (nm - 1) + ni + p2
            size = so * (no - 1) + sm * (nm - 1) + ni
            st = [0, 0, 0]
            st[perm[0]], st[perm[1]], st[perm[2]] = si, sm, so
            out.append((size, p3, st))
    return out


class Search:
    def __init__(self, D, Q, NC, E, T):
        self.D, self.Q, self.NC, self.E, self.T = D, Q, NC, E, T
        NA = 2 if NC == 3 else 1
        NR = NA
        self.ns = {"X": 1, "T1": NA, "T2": NC, "W": NC, "R": NR}
        self.ext = {"X": (D, D, D), "T1": (Q, D, D), "T2": (Q, Q, D), "W": (Q, Q, D), "R": (Q, D, D)}
        self.stage_dims = {"A": (D, D), "B": (Q, D), "C": (Q, Q), "D": (Q, D), "E": (D, D), "G": (D, D * D)}
        self.cache = {}

    def warps(self, st, m):
        n1, n2 = self.stage_dims[st]
        return thread_lines(m, self.E, self.T, n1, n2)

    def access(self, buf, side, m):
        """Instructions of the writer/reader stage of buf (per component)."""
        D, Q = self.D, self.Q
        if buf == "X":
            if side == "w":  # gather: lane (i, j + D k)
                return instrs(self.warps("G", m), lambda e, i, jk: (e, i, jk % D, jk // D), [])
            return instrs(self.warps("A", m), lambda e, j, k, i: (e, 0 * j + i, j, k), [D])
        if buf == "T1":
            if side == "w":
                return instrs(self.warps("A", m), lambda e, j, k, a: (e, 0 * j + a, j, k), [Q])
            return instrs(self.warps("B", m), lambda e, a, k, j: (e, a, 0 * a + j, k), [D])
        if buf == "T2":
            if side == "w":
                return instrs(self.warps("B", m), lambda e, a, k, b: (e, a, 0 * a + b, k), [Q])
            return instrs(self.warps("C", m), lambda e, a, b, k: (e, a, b, 0 * a + k), [D])
        if buf == "W":
            if side == "w":
                return instrs(self.warps("C", m), lambda e, a, b, k: (e, a, b, 0 * a + k), [D])
            return instrs(self.warps("D", m), lambda e, a, k, b: (e, a, 0 * a + b, k), [Q])
        if buf == "R":
            if side == "w":
                return instrs(self.warps("D", m), lambda e, a, k, j: (e, a, 0 * a + j, k), [D])
            return instrs(self.warps("E", m), lambda e, j, k, a: (e, 0 * j + a, j, k), [Q])
        raise KeyError(buf)

    def best(self, buf, mw, mr):
        key = (buf, mw, mr)
        if key in self.cache:
            return self.cache[key]
        Iw, Mw = self.access(buf, "w", mw)
        Ir, Mr = self.access(buf, "r", mr)
        ns = self.ns[buf]
        cands = layouts(self.ext[buf])
        lay = np.array([[ns * size + p3, *st] for size, p3, st in cands], np.int64)
        c = cost_many(lay, Iw, Mw) * ns + cost_many(lay, Ir, Mr) * ns
        # tie-break: smaller footprint
        sz = lay[:, 0]
        i = np.lexsort((sz, c))[0]
        size = cands[i][0]
        res = (int(c[i]) / self.E, tuple(int(v) for v in lay[i]), size)
        self.cache[key] = res
        return res

    def pa_cost(self, mc, pad=None):
        """PA data reads of stage C from the bulk-copied D (global layout, smem).
        pad None: the library's fixed element-stride padding."""
        key = ("PA", mc, pad)
        if key not in self.cache:
            self.cache[key] = self._pa_cost(mc, pad)
        return self.cache[key]

    def _pa_cost(self, mc, pad):
        Q = self.Q
        npa = 6 if self.NC == 3 else 1
        ps = ((npa * Q ** 3 + 1) // 2) * 2
        I, M = instrs(self.warps("C", mc), lambda e, a, b, c: (e, a, b, 0 * a + c), [Q])
        if pad is None:  # the fixed PA stride of the library (fk_internal.h pa_stride)
            n = ps
            while (n - Q * Q) % 16 > 1:
                n += 2
            pad = n - ps
        pads = [pad]
        lay = np.array([[ps + p, 1, Q, Q * Q] for p in pads], np.int64)
        c = cost_many(lay, I, M) * npa / self.E
        return float(c.min()), pad


def default_layout(D, Q, NC, E, ip):
    """EoLayDefault<D,Q,NC,IP> of pa_dfma_eo.cuh: maps and (se, s1, s2, s3) per buffer."""
    LS, LQ = D | 1, Q | 1
    NA = 2 if NC == 3 else 1
    X, T1, T2 = D * D * LS, NA * Q * D * LS, NC * Q * Q * LS
    W, R = NC * D * Q * LQ, NA * D * D * LQ
    if ip:
        P0, P1 = max(X, T2, W) | 1, max(T1, R) | 1
        WST, RST = P0, P1
    else:
        P0, P1 = max(X, T2, R) | 1, max(T1, W) | 1
        WST, RST = P1, P0
    maps = (0, 0, 1, 0, 0, 0)
    lay = {"X": (D * D * LS, 1, LS, D * LS), "T1": (P1, D * LS, 1, LS), "T2": (P0, LS, Q * LS, 1),
           "W": (WST, LQ, 1, Q * LQ), "R": (RST, 1, LQ, D * LQ)}
    return maps, lay


def eval_layout(S, maps, lay):
    mg, ma, mb, mc, md, me = maps
    pairs = {"X": (mg, ma), "T1": (ma, mb), "T2": (mb, mc), "W": (mc, md), "R": (md, me)}
    out = {}
    for b, (mw, mr) in pairs.items():
        Iw, Mw = S.access(b, "w", mw)
        Ir, Mr = S.access(b, "r", mr)
        l = np.array([lay[b]], np.int64)
        out[b] = (int(cost_many(l, Iw, Mw)[0]) + int(cost_many(l, Ir, Mr)[0])) * S.ns[b] / S.E
    out["PA"] = S.pa_cost(mc, 0)[0]
    return out


def cxx(name, D, Q, NC, maps, parts, ip):
    """C++ layout policy for pa_dfma_eo.cuh."""
    mg, ma, mb, mc, md, me = maps
    lines = [f"// tools/smem_strides.py {D} {Q} {NC} (E, T as instantiated)",
             f"struct {name} {{",
             f"  static constexpr bool W_OVER_T2 = {'true' if ip else 'false'};",
             f"  static constexpr int MG = {mg}, MA = {ma}, MB = {mb}, MC = {mc}, MD = {md}, ME = {me};"]
    for b in ("X", "T1", "T2", "W", "R"):
        c, (se, s1, s2, s3), size = parts[b]
        lines.append(f"  using {b} = BufLay<{se}, {size}, {s1}, {s2}, {s3}>;")
    lines.append("};")
    return "\n".join(lines)


def main():
    D, Q, NC, E, T = (int(a) for a in sys.argv[1:6])
    S = Search(D, Q, NC, E, T)
    for ip in (False, True):
        maps, lay = default_layout(D, Q, NC, E, ip)
        ev = eval_layout(S, maps, lay)
        print(f"default layout (IP={ip}): {sum(ev.values()):.1f} wf/elem  " +
              " ".join(f"{k} {v:.1f}" for k, v in ev.items()))
    res = []
    for mg, ma, mb, mc, md, me in itertools.product((0, 2), MAPS, MAPS, MAPS, MAPS, MAPS):
        parts = {"X": S.best("X", mg, ma), "T1": S.best("T1", ma, mb), "T2": S.best("T2", mb, mc),
                 "W": S.best("W", mc, md), "R": S.best("R", md, me)}
        tot = sum(p[0] for p in parts.values()) + S.pa_cost(mc)[0]
        res.append((tot, (mg, ma, mb, mc, md, me), parts))
    res.sort(key=lambda r: r[0])
    base = res[[r[1] for r in res].index((0, 0, 0, 0, 0, 0))]
    print(f"all maps 0: {base[0]:.1f} wf/elem")
    print(cxx(f"EoLay_d{D}q{Q}c{NC}e{E}", D, Q, NC, res[0][1], res[0][2], "--ip" in sys.argv))
    for tot, maps, parts in res[:3]:
        print(f"maps G,A,B,C,D,E = {maps}: {tot:.1f} wf/elem  PA (cost, pad) {S.pa_cost(maps[3])}")
        for k, (c, lay, size) in parts.items():
            print(f"    {k:3s} {c:6.1f} wf/el  (se, s1, s2, s3) = {lay}  comp size {size}")


if __name__ == "__main__":
    main()
