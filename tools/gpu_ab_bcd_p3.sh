for i in 1 2; do
  for c in 49 51 52 50; do
    v=$(FK_CFG=$c timeout 300 python bench.py --p 3 --n 71 --kind mass --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['impl_config']['cfg'])")
    echo "p 3 rep $i cfg $c: $v"
  done
  for c in 0 4; do
    v=$(FK_MIX_CFG=$c timeout 300 python bench.py --mixed --p 8 --n 40 --steps 30 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3))")
    echo "mixed p 8 rep $i cfg $c: $v"
  done
done
