# p=4 geometry check: parity of the new cfgs, then a repeated p=4 sweep (3 reps) for noise
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "launch_config and eo-19 or launch_config and eo-20" 2>&1 | tail -2
for r in 1 2 3; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_p4_r$r.jsonl \
  --sweep-kinds diffusion --sweep-orders 4 --sweep-cfgs eo1,eo2,eo5,eo6,eo10,eo14,eo19,eo20,mf5 > /dev/null 2>&1
python tools/sweep_table.py gpurun_out/sweep_p4_r$r.jsonl | tail -1
done
