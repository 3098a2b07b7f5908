# Full round-end style GPU pass: smoke, gpu tests, bench, CG configs, ncu launch list + full capture.
set -x
tag=${1:-r}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_$tag.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 | tee gpurun_out/bench_ref_$tag.json
timeout 600 python bench.py --cg weak 2>&1 | tail -1 | tee gpurun_out/cg_weak_$tag.json
timeout 900 python bench.py --cg strong 2>&1 | tail -1 | tee gpurun_out/cg_strong_$tag.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
