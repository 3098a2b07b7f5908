set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_r17_bp1p4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --kind mass --p 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pa_pipe -s 3 -c 1 -o gpurun_out/prof_r17_bp3p8 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --p 8 > /dev/null 2>&1
ls gpurun_out/
