"""Print the FK_VARIANT_AUTO table (fk_api.cu kAutoVar*/kAutoCfg*) from a sweep
JSONL file: the fastest (variant, cfg) per (kind, p).

    python tools/auto_table.py profiles/r01_sweep_vNN.jsonl
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
rows = [r for r in rows if r["variant"] != "mf"]  # the PA table (MF has its own, kAutoCfgMF*)
code = {"dfma": "D_", "dmma": "M_", "eo": "O_"}
for kind, nc in (("diffusion", 3), ("mass", 1)):
    var, cfg = ["D_"], [0]
    for p in range(1, 9):
        sel = [r for r in rows if r["kind"] == kind and r["p"] == p]
        b = max(sel, key=lambda r: r["gdofs"])
        var.append(code[b["variant"]])
        cfg.append(b["cfg"])
        print(f"// {kind} p={p}: {b['variant']}{b['cfg']} {b['gdofs']:.2f} GDOF/s ({b['hbm_frac']:.2f} HBM)",
              file=sys.stderr)
    print(f"const int kAutoVar{nc}[9] = {{{', '.join(var)}}};")
    print(f"const int kAutoCfg{nc}[9] = {{{', '.join(map(str, cfg))}}};")
