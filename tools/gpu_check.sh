set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 2>&1 | tail -3 | tee gpurun_out/bench1.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pa_dfma -c 5 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_dfma -s 3 -c 1 -o gpurun_out/prof1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
