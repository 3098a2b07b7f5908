# Final per-order table: the auto-selected default (FK_VARIANT_AUTO) for BP3
# and BP1 at p = 1..8 on the ~10 M-dof sweep meshes, 200 applies each.
for kind in diffusion mass; do
  for p in 1 2 3 4 5 6 7 8; do
    case $p in 1) n=214;; 2) n=107;; 3) n=71;; 4) n=54;; 5) n=43;; 6) n=36;; 7) n=31;; 8) n=27;; esac
    timeout 300 python bench.py --p $p --n $n --kind $kind --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(json.dumps({'kind': '$kind', 'p': $p, 'n': $n, 'gdofs': round(d['value'],2), 'kernel_frac': round(r['frac'],3), 'variant': d['impl_config']['variant'], 'cfg': d['impl_config']['cfg'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))"
  done
done
