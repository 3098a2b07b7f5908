# Searched smem layouts: parity of every geometry, then the sweep (both kinds, all orders).
set -x
tag=${1:-eolay}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_${tag}.jsonl \
  --sweep-cfgs dfma0,dfma2,dfma6,eo0,eo1,eo2,eo3,eo4,eo5,eo6,eo7,eo8,eo9,eo10,eo11,eo12,eo13,eo14,eo15,eo16,eo17,eo18 > /dev/null 2> gpurun_out/sweep_${tag}.log
python tools/sweep_table.py gpurun_out/sweep_${tag}.jsonl
