# ncu --set full of the fused kernel for given (variant, cfg) pairs at BP3 p (default 4).
# usage: bash tools/gpu_ncu_cfg.sh TAG P variant:cfg [variant:cfg ...]
tag=$1; p=$2; shift 2
for vc in "$@"; do
  v=${vc%%:*}; c=${vc##*:}
  FK_CFG=$c timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 \
    -o gpurun_out/ncu_${tag}_p${p}_${v}${c} python bench.py --p $p --kind ${KIND:-diffusion} --variant $v --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_${tag}_p${p}_${v}${c}.log 2>&1
  tail -1 gpurun_out/ncu_${tag}_p${p}_${v}${c}.log
done
