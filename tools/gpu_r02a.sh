set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
python tools/make_psi_fixtures.py C2 C3 C4 C5 --out tests/golden > gpurun_out/r02a/fixtures.log 2>&1
cp tests/golden/psi_*.npz gpurun_out/r02a/
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02a/pytest_gpu.txt 2>&1
timeout 1800 python tools/parity_census.py c2 c2c c3c c5c c3 c5 c4 c4c c1c --mode both > gpurun_out/r02a/census.txt 2>&1
echo done
