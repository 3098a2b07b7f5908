timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_dh.jsonl --sweep-orders 2,4,6,8 \
  --sweep-cfgs eo2,eo10,eo14,eo18,eo19,eo25,eo26,eo27 > /dev/null 2>&1
python tools/sweep_table.py gpurun_out/sweep_dh.jsonl
python -c "
import json
for l in open('gpurun_out/sweep_dh.jsonl'):
    r=json.loads(l)
    if r['cfg'] in (10,14,25,26,27) and r['kind']=='diffusion': print(r['p'], r['cfg'], round(r['gdofs'],2), r['launch'])
"
