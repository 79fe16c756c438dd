# Re-entry check of the current tree: full GPU tests, default bench line, C3/C5 kernel timings.
set -x
T=${1:-r02h}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.log 2>&1; tail -n 1 $O/bench.log > $O/bench_c4.json
for c in C3 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton --no-hbm > $O/bench_$c.json 2> $O/bench_$c.err
done
tail -3 $O/pytest_gpu.txt; cat $O/bench_c4.json
