#!/bin/bash
# Round-end measurement set (run under gpurun): bench line, launch list, ncu
# metrics of the cell kernels on one bench step, full captures of the two
# dominant kernels.  usage: bash tools/round_profile.sh TAG
T=${1:-rXX}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.log 2>&1; tail -1 gpurun_out/${T}_bench.log > gpurun_out/${T}_bench_c4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio
PF_NCU_STEP=1 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_kernels_metrics.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
for k in k_cells_build k_cells_eval_sync; do
  PF_NCU_STEP=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/${T}_${k}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
ls -la gpurun_out/ | grep $T
