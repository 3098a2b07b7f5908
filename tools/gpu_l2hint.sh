timeout 900 python -m pytest tests -m gpu -q -x -k "launch_config and (eo or mf)" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | head -c 200; echo; done
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_l2h.jsonl --sweep-kinds diffusion \
  --sweep-cfgs eo1,eo2,eo5,eo10,eo11,eo14,eo18 > /dev/null 2>&1
python tools/sweep_table.py gpurun_out/sweep_l2h.jsonl
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pa_pipe -s 5 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__|duration|hit_rate"
