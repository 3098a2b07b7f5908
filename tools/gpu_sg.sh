timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_sg.jsonl \
  --sweep-cfgs eo1,eo2,eo5,eo10,eo11,eo14,eo18,eo19,eo20,eo21,eo22,eo23,eo24 > /dev/null 2>&1
python tools/sweep_table.py gpurun_out/sweep_sg.jsonl
