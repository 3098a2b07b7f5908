# default bench (sustained + burst), launch list and one ncu --set full of the default kernel
tag=${1:-def}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_$tag.json
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_short_$tag.json
timeout 600 python bench.py --kind mass --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_bp1_$tag.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/ncu_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in bench bench_short bench_bp1; do echo "$f: $(head -c 400 gpurun_out/${f}_$tag.json)"; done
