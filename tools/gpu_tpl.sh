set -x
tag=${1:-tpl}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_${tag}.jsonl \
  --sweep-cfgs dfma0,dfma6,eo1,eo2,eo5,eo6,eo9,eo10,eo11,eo14,eo15,eo18,eo19,eo20,eo21,eo22 --sweep-orders 1,2,3,4 > /dev/null 2> gpurun_out/sweep_${tag}.log
python tools/sweep_table.py gpurun_out/sweep_${tag}.jsonl
