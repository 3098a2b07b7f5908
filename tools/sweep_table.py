"""Pivot a bench.py --sweep JSONL file: GDOF/s per (kind, p) x (variant, cfg)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
cols = sorted({(r["variant"], r["cfg"]) for r in rows})
print("kind  p  " + " ".join(f"{v}{c:<6}" for v, c in cols) + "  best(hbm)")
for kind in ("diffusion", "mass"):
    for p in range(1, 9):
        sel = {(r["variant"], r["cfg"]): r for r in rows if r["kind"] == kind and r["p"] == p}
        if not sel:
            continue
        best = max(sel.values(), key=lambda r: r["gdofs"])
        print(f"{kind[:4]} {p}  " + " ".join(f"{sel[c]['gdofs']:10.2f}" if c in sel else " " * 10 for c in cols)
              + f"  {best['variant']}{best['cfg']} {best['hbm_frac']:.2f}")
