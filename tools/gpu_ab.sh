# A/B of launch configs on the default bench (alternating, repeated):
#   bash tools/gpu_ab.sh "29 32" [reps] [steps] [extra bench args]
cfgs=$1; reps=${2:-3}; steps=${3:-200}; shift 3
for i in $(seq $reps); do
  for c in $cfgs; do
    v=$(FK_CFG=$c timeout 300 python bench.py --steps $steps --warmup 10 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])")
    echo "rep $i cfg $c: $v"
  done
done
