# Per-order ncu counters, DMMA vs the even-odd FMA kernel (BP3, SWEEP_N meshes):
# FP64 pipe and DMMA sub-pipe utilisation, DRAM bytes, time, instructions, smem wavefronts.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
out=gpurun_out/ncu_orders.csv
: > $out
for spec in "1 dmma 2" "1 eo 1" "2 dmma 2" "2 eo 1" "3 dmma 2" "3 eo 2" "4 dmma 2" "4 eo 5" "5 dmma 2" "5 eo 2" "6 dmma 2" "6 eo 14" "7 dmma 2" "7 eo 18" "8 dmma 2" "8 eo 10"; do
  set -- $spec
  FK_CFG=$3 timeout 300 ncu --metrics $M --clock-control none -k regex:pa_pipe -s 3 -c 1 --csv python bench.py --p $1 --variant $2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -v "^==" | sed "s/^/$1,$2,$3,/" >> $out
done
wc -l $out
