# Block operator: default launch config per order vs the single-X (8-11) and
# YS+SX (12-15) twins, 30 applies, 2 reps, ~130 M dofs per order; FusedMF at
# order 4 on the paper's 128^3 configuration.
declare -A C=([2]="0 8 12" [3]="3 11 0 8" [4]="2 10 14 6" [5]="2 10 14" [6]="0 8 12" [7]="0 8 12" [8]="4 8 12")
for i in 1 2; do
  for p in 2 3 4 5 6 7 8; do
    case $p in 2) n=160;; 3) n=110;; 4) n=80;; 5) n=64;; 6) n=54;; 7) n=46;; 8) n=40;; esac
    for c in ${C[$p]}; do
      v=$(FK_MIX_CFG=$c timeout 300 python bench.py --mixed --p $p --n $n --steps 30 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3))")
      echo "order $p rep $i cfg $c: $v"
    done
  done
  for c in 2 10; do
    v=$(FK_MIX_CFG=$c timeout 300 python bench.py --mixed --variant mf --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2))")
    echo "FusedMF order 4 128^3 rep $i cfg $c: $v"
  done
  for c in 2 10; do
    v=$(FK_MIX_CFG=$c timeout 300 python bench.py --mixed --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3))")
    echo "FusedPA order 4 128^3 rep $i cfg $c: $v"
  done
done
