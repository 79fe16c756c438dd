set -x
mkdir -p gpurun_out/r02b
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02b/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b/bench_ref.json 2> gpurun_out/r02b/bench_ref.err
echo done
