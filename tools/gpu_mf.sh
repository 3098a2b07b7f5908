set -x
tag=${1:-mf}
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_${tag}.jsonl \
  --sweep-cfgs eo1,mf0,mf1,mf2,mf3,mf4,mf5,mf6,mf7 > /dev/null 2> gpurun_out/sweep_${tag}.log
python tools/sweep_table.py gpurun_out/sweep_${tag}.jsonl
