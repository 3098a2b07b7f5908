# Mixed-operator launch-geometry sweep: order_p 2..8 x FK_MIX_CFG (default 0..3), ~130 M dofs each.
tag=${1:-mix}
out=gpurun_out/mixsweep_${tag}.jsonl
: > $out
for p in 2 3 4 5 6 7 8; do
  case $p in 2) n=160;; 3) n=110;; 4) n=80;; 5) n=64;; 6) n=54;; 7) n=46;; 8) n=40;; esac
  for c in ${CFGS:-0 1 2 3}; do
    FK_MIX_CFG=$c timeout 300 python bench.py --mixed --p $p --n $n --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); d['p']=$p; d['cfg']=$c; print(json.dumps(d))" >> $out
  done
done
python -c "
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['p'], d['cfg'], round(d['value'],2), round(d['roofline']['frac'],3), d['config']['launch'], round(d['rk4_gdofs_per_apply'],2))
" $out
