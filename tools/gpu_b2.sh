for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b2_$i.json; done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b2_short.json
