# A/B of two builds of libfk_b200.so on one box: alternating bench runs.
#   bash tools/gpu_ab_lib.sh VARIANT_LIB "bench args" ROUNDS
v=$1; args=$2; n=${3:-3}
for r in $(seq 1 $n); do
  a=$(python bench.py $args --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f %.4f' % (d['value'], d['roofline']['kernel_ms']))")
  b=$(FK_LIB_PATH=$v python bench.py $args --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f %.4f' % (d['value'], d['roofline']['kernel_ms']))")
  echo "[$args] round $r: product $a | variant $b"
done
