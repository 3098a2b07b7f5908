# Round-2 evidence pass: smoke, bench (driver K/W) + reference arm, CG, mixed,
# MF, deterministic, launch lists, one full ncu capture of the default kernel.
set -x
tag=${1:-r02}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -4 gpurun_out/smoke_$tag.log
timeout 600 python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_$tag.json
timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench1000_$tag.json
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_ref_$tag.json
timeout 600 python bench.py --cg weak --cpu-seconds 8 2>/dev/null | tail -1 > gpurun_out/cg_weak_$tag.json
timeout 900 python bench.py --cg strong --cpu-seconds 8 2>/dev/null | tail -1 > gpurun_out/cg_strong_$tag.json
timeout 600 python bench.py --cg weak --variant mf --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/cg_weak_mf_$tag.json
timeout 900 python bench.py --cg strong --variant mf --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/cg_strong_mf_$tag.json
timeout 600 python bench.py --mixed --steps 20 --warmup 3 2>/dev/null | tail -1 > gpurun_out/mixed_$tag.json
timeout 600 python bench.py --variant mf --steps 200 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_mf_$tag.json
timeout 600 python bench.py --deterministic --steps 200 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_det_$tag.json
timeout 300 env FK_BENCH_DEVICE=0 python bench.py --gpus 2 --n 24 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_2rank_shared_$tag.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cg_$tag.csv python bench.py --cg weak --no-cpu-baseline > /dev/null 2>&1
for f in bench bench1000 bench_ref cg_weak cg_strong cg_weak_mf cg_strong_mf mixed bench_mf bench_det bench_2rank_shared; do echo "$f: $(head -c 260 gpurun_out/${f}_$tag.json)"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 5 -c 1 -o gpurun_out/ncu_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/ncu_$tag.ncu-rep
python tools/ncu_summary.py gpurun_out/ncu_$tag.ncu-rep > gpurun_out/ncu_${tag}_summary.json; rm -f gpurun_out/ncu_$tag.ncu-rep
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sweep gpurun_out/sweep_$tag.jsonl > /dev/null 2>&1; wc -l gpurun_out/sweep_$tag.jsonl
