# ncu full capture of the fused kernel: tools/gpu_prof2.sh TAG P VARIANT [N]
set -x
tag=$1; p=$2; v=$3; n=${4:-}
extra=""; [ -n "$n" ] && extra="--n $n"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_${tag}_p${p}_$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --variant $v --p $p $extra > gpurun_out/ncu_${tag}_p${p}_$v.log 2>&1
tail -1 gpurun_out/ncu_${tag}_p${p}_$v.log
