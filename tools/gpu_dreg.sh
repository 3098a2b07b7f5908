# DM_REG evaluation: parity of every launch geometry (incl. multi-batch), then a focused sweep.
set -x
tag=${1:-dreg}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_${tag}_bp3.jsonl \
  --sweep-kinds diffusion --sweep-cfgs eo0,eo2,eo4,eo5,eo6,eo9,eo10,eo11,dfma0,dfma2,dfma7,dfma8 > /dev/null 2> gpurun_out/sweep_${tag}_bp3.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_${tag}_bp1.jsonl \
  --sweep-kinds mass --sweep-cfgs eo0,eo1,eo5,eo8,eo9,eo10,eo11,dfma6,dfma7,dfma8 > /dev/null 2> gpurun_out/sweep_${tag}_bp1.log
python tools/sweep_table.py gpurun_out/sweep_${tag}_bp3.jsonl
python tools/sweep_table.py gpurun_out/sweep_${tag}_bp1.jsonl
