# parity of every launch config + a focused sweep after a kernel change
tag=${1:-xpre}
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_$tag.jsonl \
  --sweep-cfgs ${CFGS:-eo2,eo10,eo14,eo18,eo19,eo23,eo24,mf4,mf5,mf6} > /dev/null 2>&1
python tools/sweep_table.py gpurun_out/sweep_$tag.jsonl
