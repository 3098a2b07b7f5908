"""Shared-memory wavefront model of the DFMA line kernel (design-time aid).

Counts 128-byte wavefronts for every 8-byte LDS/STS the stage loops of
pa_dfma.cuh issue for one CTA batch, given the line pitches (LS, LQ) and
the per-element region strides (P0, P1, XS).  An 8-byte warp access is
split into two half-warps; within a half-warp the wavefront count is the
maximum number of distinct 8-byte words that fall into the same bank pair
(32 x 4-byte banks = 16 x 8-byte bank pairs), same-word requests broadcast.

    python tools/smem_model.py 5 6 3 4 96 2      # D Q NC E T NL
    python tools/smem_model.py 5 6 3 4 96 2 --search
"""

from __future__ import annotations

import itertools
import sys


def wavefronts(addrs):
    """addrs: list (len <= 32) of 8-byte word addresses (None = inactive lane)."""
    total = 0
    for half in (addrs[:16], addrs[16:]):
        words = {a for a in half if a is not None}
        if not words:
            continue
        per_bank = {}
        for w in words:
            per_bank.setdefault(w % 16, set()).add(w)
        total += max(len(s) for s in per_bank.values())
    return total


def ideal(addrs):
    total = 0
    for half in (addrs[:16], addrs[16:]):
        if any(a is not None for a in half):
            total += 1
    return total


def stage_accesses(D, Q, NC, E, T, NL, LS, LQ, P0, P1, XS):
    """Yield (name, list_of_warp_accesses); each warp access = 32 word addresses."""
    NA = 2 if NC == 3 else 1
    NR = 2 if NC == 3 else 1
    S0, S1, SX = 0, 100000, 200000  # separate regions (different arrays)

    def lines(n, nl):
        """per warp-iteration: list of lane->line (None)"""
        out = []
        for t0 in range(0, n, nl * T):
            for h in range(nl):
                for w0 in range(0, T, 32):
                    lanes = []
                    for l in range(32):
                        t = t0 + h * T + w0 + l
                        lanes.append(t if (w0 + l < T and t < n) else None)
                    if any(x is not None for x in lanes):
                        out.append(lanes)
        return out

    acc = []
    ne = E
    # stage A: read X[e][v*LS + i], write T1 at (v//D)*LS + v%D + a*D*LS (+ s)
    for lanes in lines(ne * D * D, NL):
        for i in range(D):
            acc.append(("A.ld", [None if t is None else SX + (t // (D * D)) * XS + (t % (D * D)) * LS + i for t in lanes]))
        for s in range(NA):
            for a in range(Q):
                acc.append(("A.st", [None if t is None else S1 + (t // (D * D)) * P1 + s * Q * D * LS + a * D * LS
                                     + ((t % (D * D)) // D) * LS + (t % (D * D)) % D for t in lanes]))
    # stage B: read T1 u*LS + j (+ s*Q*D*LS), write T2 s*Q*Q*LS + b*Q*LS + a*LS + k
    for lanes in lines(ne * D * Q, NL):
        for s in range(NA):
            for j in range(D):
                acc.append(("B.ld", [None if t is None else S1 + (t // (D * Q)) * P1 + s * Q * D * LS + (t % (D * Q)) * LS + j for t in lanes]))
        for s in range(NC):
            for b in range(Q):
                acc.append(("B.st", [None if t is None else S0 + (t // (D * Q)) * P0 + s * Q * Q * LS + b * Q * LS
                                     + ((t % (D * Q)) // D) * LS + (t % (D * Q)) % D for t in lanes]))
    # stage C: read T2 r*LS + k, write W s*D*Q*LQ + k*Q*LQ + a*LQ + b  (r = a + Q b)
    nlc = 1 if (NC == 3 and 6 * D * NL > 60) else NL
    for lanes in lines(ne * Q * Q, nlc):
        for s in range(NC):
            for k in range(D):
                acc.append(("C.ld", [None if t is None else S0 + (t // (Q * Q)) * P0 + s * Q * Q * LS + (t % (Q * Q)) * LS + k for t in lanes]))
        for s in range(NC):
            for k in range(D):
                acc.append(("C.st", [None if t is None else S1 + (t // (Q * Q)) * P1 + s * D * Q * LQ + k * Q * LQ
                                     + ((t % (Q * Q)) % Q) * LQ + (t % (Q * Q)) // Q for t in lanes]))
    # stage D: read W u*LQ + b (+ s*D*Q*LQ), write R s*D*D*LQ + (k*D + j)*LQ + a   (u = a + Q k)
    for lanes in lines(ne * Q * D, NL):
        for s in range(NC):
            for b in range(Q):
                acc.append(("D.ld", [None if t is None else S1 + (t // (Q * D)) * P1 + s * D * Q * LQ + (t % (Q * D)) * LQ + b for t in lanes]))
        for s in range(NR):
            for j in range(D):
                acc.append(("D.st", [None if t is None else S0 + (t // (Q * D)) * P0 + s * D * D * LQ
                                     + ((t % (Q * D)) // Q) * D * LQ + j * LQ + (t % (Q * D)) % Q for t in lanes]))
    # stage E: read R v*LQ + a (+ s*D*D*LQ)
    for lanes in lines(ne * D * D, NL):
        for s in range(NR):
            for a in range(Q):
                acc.append(("E.ld", [None if t is None else S0 + (t // (D * D)) * P0 + s * D * D * LQ + (t % (D * D)) * LQ + a for t in lanes]))
    return acc


def cost(D, Q, NC, E, T, NL, LS, LQ, P0, P1, XS, detail=False):
    tot = idl = 0
    per = {}
    for name, addrs in stage_accesses(D, Q, NC, E, T, NL, LS, LQ, P0, P1, XS):
        w, i = wavefronts(addrs), ideal(addrs)
        tot += w
        idl += i
        p = per.setdefault(name, [0, 0])
        p[0] += w
        p[1] += i
    if detail:
        for k, (w, i) in sorted(per.items()):
            print(f"  {k}: {w / E:7.1f} wf/elem (ideal {i / E:6.1f})")
    return tot / E, idl / E


def sizes(D, Q, NC, LS, LQ):
    NA = 2 if NC == 3 else 1
    NR = 2 if NC == 3 else 1
    p0 = max(NC * Q * Q * LS, NR * D * D * LQ)
    p1 = max(NA * Q * D * LS, NC * D * Q * LQ)
    return p0, p1, D * D * LS


def main():
    D, Q, NC, E, T, NL = (int(a) for a in sys.argv[1:7])
    LS, LQ = D | 1, Q | 1
    p0, p1, xs = sizes(D, Q, NC, LS, LQ)
    P0, P1 = p0 | 1, p1 | 1
    c, i = cost(D, Q, NC, E, T, NL, LS, LQ, P0, P1, xs, detail=True)
    print(f"current LS={LS} LQ={LQ} P0={P0} P1={P1}: {c:.1f} wf/elem (ideal {i:.1f})")
    if "--search" in sys.argv:
        best = []
        for ls, lq in itertools.product(range(D, D + 9), range(Q, Q + 9)):
            p0, p1, xs = sizes(D, Q, NC, ls, lq)
            for d0, d1 in itertools.product(range(0, 9), range(0, 9)):
                c, _ = cost(D, Q, NC, E, T, NL, ls, lq, p0 + d0, p1 + d1, xs)
                best.append((c, ls, lq, p0 + d0, p1 + d1, (p0 + d0 + p1 + d1) * E * 8))
        best.sort()
        for b in best[:8]:
            print("  wf/elem %.1f  LS=%d LQ=%d P0=%d P1=%d smem=%d B" % b)


if __name__ == "__main__":
    main()
