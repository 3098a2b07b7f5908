# BP3 p=4 (54^3) top geometries under the default bench's sustained load
# (1000 applies, power-capped clocks), 2 reps, interleaved.
for i in 1 2; do
  for c in 35 29 32 25 1 2 11 14 41 45; do
    v=$(FK_CFG=$c timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['impl_config']['cfg'])")
    echo "rep $i cfg $c: $v"
  done
done
