# 200-apply A/B: BP1 p = 1, 2 defaults vs the thread-per-element kernel (cfgs 58, 59)
for i in 1 2; do
  for p in 1 2; do
    case $p in 1) n=214; cs="${CS1:-24 58 59}";; 2) n=107; cs="${CS2:-31 58 59}";; esac
    for c in $cs; do
      v=$(FK_CFG=$c timeout 300 python bench.py --p $p --n $n --kind mass --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['impl_config']['cfg'], d['clocks']['sm_mhz'])")
      echo "p $p rep $i cfg $c: $v"
    done
  done
done
