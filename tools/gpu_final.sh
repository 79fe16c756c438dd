# Round-end evidence set (one gpurun call): tests, smoke, bench lines (C4 headline + C2/C3/C5),
# reference arm, parity census, launch list, per-kernel ncu metrics, full captures of the two
# cell kernels, HBM kernels (grid, PCG, kNN) under ncu.   usage: bash tools/gpu_final.sh TAG
set -x
T=${1:-final}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.log 2>&1; tail -n 1 $O/bench.log > $O/bench_c4.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; tail -n 1 $O/bench_ref.log > $O/bench_reference_c4.json
for c in C2 C3 C5; do
  timeout 900 python bench.py --config $c --no-cpu > $O/bench_$c.log 2>&1; tail -n 1 $O/bench_$c.log > $O/bench_$c.json
done
timeout 1800 python tools/parity_census.py c2 c2c c3c c5c c3 c5 c4 c4c c1c --mode both > $O/census.txt 2>&1
python tools/hbm_probe.py C4 > $O/hbm_probe.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    --log-file $O/hbm_kernels.csv python tools/hbm_probe.py C4 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
PF_NCU_STEP=1 timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/kernels_metrics.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-newton --no-hbm > /dev/null 2>&1
for k in k_cells_build k_cells_eval_sync; do
  PF_NCU_STEP=1 timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o $O/${k}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-newton --no-hbm > /dev/null 2>&1
done
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:k_pcg_sell -c 1 -o $O/pcg_full python tools/hbm_probe.py C4 > /dev/null 2>&1
ls -la $O
