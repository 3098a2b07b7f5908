# ncu full captures of the fused kernel for given variants at p=4 (BP3 54^3)
set -x
tag=${1:-r}
shift
for v in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_${tag}_$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/ncu_${tag}_$v.log 2>&1
  tail -1 gpurun_out/ncu_${tag}_$v.log
done
