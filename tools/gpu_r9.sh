set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_r9.jsonl > /dev/null 2> gpurun_out/sweep_r9.log
bash tools/gpu_prof.sh r9 dmma
