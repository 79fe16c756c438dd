mkdir -p gpurun_out/q9
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fluid.py -q -x -p no:cacheprovider > gpurun_out/q9/pytest.txt 2>&1
python tools/hbm_probe.py C4 > gpurun_out/q9/hbm_probe.json 2>&1
python tools/hbm_probe.py C3 > gpurun_out/q9/hbm_probe_c3.json 2>&1
tail -n 3 gpurun_out/q9/pytest.txt; cat gpurun_out/q9/hbm_probe.json gpurun_out/q9/hbm_probe_c3.json
