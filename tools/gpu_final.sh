# Round-end style pass: smoke, all GPU tests, bench (+ reference arm), CG, mixed, MF, sweep, launch list.
set -x
tag=${1:-fin}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_$tag.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref_$tag.json
timeout 600 python bench.py --cg weak 2>&1 | tail -1 > gpurun_out/cg_weak_$tag.json
timeout 900 python bench.py --cg strong 2>&1 | tail -1 > gpurun_out/cg_strong_$tag.json
timeout 600 python bench.py --mixed --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/mixed_$tag.json
timeout 600 python bench.py --mixed --variant mf --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/mixed_mf_$tag.json
timeout 600 python bench.py --variant mf --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_mf_$tag.json
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_$tag.jsonl > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in bench bench_ref cg_weak cg_strong mixed mixed_mf bench_mf; do echo "$f: $(head -c 300 gpurun_out/${f}_$tag.json)"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/ncu_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
