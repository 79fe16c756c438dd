set -x
T=r02g
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist_plane.py tests/test_gpu_dist_newton.py -q -x -p no:cacheprovider > $O/pytest_dist.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
python tools/hbm_probe.py C4 > $O/hbm_probe.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    --log-file $O/hbm_kernels.csv python tools/hbm_probe.py C4 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:k_grid_coop -c 1 -o $O/grid_full python tools/hbm_probe.py C4 > /dev/null 2>&1
tail -3 $O/pytest_dist.txt $O/pytest_gpu.txt; cat $O/hbm_probe.json
