mkdir -p gpurun_out/q10
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_build.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/q10/pytest.txt 2>&1
for rep in 1 2; do for e in 0 1; do for c in C4 C3 C5; do
  PF_EVAL_SORT=$e timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton --no-hbm > gpurun_out/q10/b_${e}_${c}_$rep.json 2>/dev/null
  echo "sort=$e $c rep$rep $(python -c "import json;d=json.loads(open('gpurun_out/q10/b_${e}_${c}_$rep.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), round(d['roofline']['split']['eval_ms'],2))")"
done; done; done > gpurun_out/q10/summary.txt
tail -n 2 gpurun_out/q10/pytest.txt; cat gpurun_out/q10/summary.txt
