# full GPU test suite + C4 bench (kernel-only) + HBM kernels under ncu
T=${1:-check}
O=gpurun_out/$T
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton > $O/bench_c4.json 2> $O/bench_c4.err
python tools/hbm_probe.py C4 > $O/hbm_probe.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    --log-file $O/hbm_kernels.csv python tools/hbm_probe.py C4 > /dev/null 2>&1
tail -3 $O/pytest_gpu.txt; cat $O/hbm_probe.json
python -c "import json;d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], json.dumps(d.get('roofline_hbm_kernels'))[:900])"
