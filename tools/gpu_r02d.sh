set -x
T=r02d
O=gpurun_out/$T
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.txt 2>&1
python tools/hbm_probe.py C4 > $O/hbm_probe.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/hbm_kernels.csv python tools/hbm_probe.py C4 > $O/hbm_probe_ncu.json 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench.json 2> $O/bench.err
ls -la $O
