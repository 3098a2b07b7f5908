# usage: bash tools/gpu_ab_orders.sh "cfg cfg ..."  (BP3, or KIND=mass, at ORDERS (default 5 6 7 3) on the sweep meshes, 200 applies, 2 reps)
for p in ${ORDERS:-5 6 7 3}; do
  case $p in 1) n=214;; 2) n=107;; 3) n=71;; 4) n=54;; 5) n=43;; 6) n=36;; 7) n=31;; 8) n=27;; esac
  for i in 1 2; do
    for c in $1; do
      v=$(FK_CFG=$c timeout 300 python bench.py --p $p --n $n --steps 200 --warmup 10 --no-cpu-baseline ${KIND:+--kind $KIND} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3))")
      echo "p $p rep $i cfg $c: $v"
    done
  done
done
