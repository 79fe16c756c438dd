# Full ncu captures (with source) of the two fast-tier cell kernels on one C4 bench step.
# usage: bash tools/gpu_ncu_cells.sh TAG [CONFIG]
T=${1:-ncu}; CFG=${2:-C4}
O=gpurun_out/$T
mkdir -p $O
for k in k_cells_build k_cells_eval_sync; do
  PF_NCU_STEP=1 timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o $O/${k}_${CFG} python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu --no-newton --no-hbm > $O/${k}_${CFG}.log 2>&1
done
ls -la $O
