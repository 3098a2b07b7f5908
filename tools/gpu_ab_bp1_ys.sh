# 200-apply A/B of the BP1 default cfg per order against the staged-scatter
# candidates (cfgs 40-49), 2 reps, on the sweep meshes.
declare -A C=([2]="24 31 44 49" [3]="24 31 44 49 40" [4]="30 40 41 46 47" [5]="35 41 47 40" [6]="30 41 47 45" [7]="23 42 43 41 47" [8]="30 41 45 42")
for p in 2 3 4 5 6 7 8; do
  case $p in 1) n=214;; 2) n=107;; 3) n=71;; 4) n=54;; 5) n=43;; 6) n=36;; 7) n=31;; 8) n=27;; esac
  for i in 1 2; do
    for c in ${C[$p]}; do
      v=$(FK_CFG=$c timeout 300 python bench.py --p $p --n $n --kind mass --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['impl_config']['cfg'])")
      echo "p $p rep $i cfg $c: $v"
    done
  done
done
