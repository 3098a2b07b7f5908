set -x
tag=${1:-r}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_$tag.jsonl > gpurun_out/bench_sweep_$tag.json 2> gpurun_out/sweep_$tag.log
tail -3 gpurun_out/sweep_$tag.log
