# quick build-kernel iteration: parity tests of the cell path + C4/C3/C5 kernel timings (no e2e/cpu/newton)
T=${1:-quick}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_build.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1
for c in C4 C3 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton --no-hbm > $O/bench_$c.json 2> $O/bench_$c.err
done
O=$O python - <<'PY' > $O/summary.txt
import json, os
O = os.environ["O"]
for c in ("C4", "C3", "C5"):
    try:
        d = json.loads(open(f"{O}/bench_{c}.json").read().strip().splitlines()[-1])
        print(c, round(d["ms_per_step"], 2), "ms", d.get("other_restriction_ms_per_step"))
    except Exception as e:
        print(c, "ERR", e)
PY
tail -1 $O/pytest.txt >> $O/summary.txt
cat $O/summary.txt
