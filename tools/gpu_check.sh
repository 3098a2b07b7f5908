# one GPU call: smoke, gpu tests, bench, sweep, ncu launch list + full capture of the top kernel
set -x
tag=${1:-r}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 2>&1 | tail -1 | tee gpurun_out/bench_$tag.json
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_$tag.jsonl > /dev/null 2> gpurun_out/sweep_$tag.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pa_pipe -c 5 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
