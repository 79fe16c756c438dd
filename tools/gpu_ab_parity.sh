# In-place build: parity tests of the cell path on the default library, then C4/C3/C5 timings of
# the build-workspace variants (variants/*.so) alternating twice.
T=${1:-ipab}; shift
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_build.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1
for rep in 1 2; do
  for v in "$@"; do
    for c in C4 C3 C5; do
      PF_LIB_PATH=variants/$v.so timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton --no-hbm \
        > $O/${v}_${c}_$rep.json 2> $O/${v}_${c}_$rep.err
    done
  done
done
O=$O python - "$@" <<'PY' > $O/summary.txt
import json, os, sys
O = os.environ["O"]
for v in sys.argv[1:]:
    row = [v]
    for c in ("C4", "C3", "C5"):
        ms = []
        for rep in (1, 2):
            try:
                d = json.loads(open(f"{O}/{v}_{c}_{rep}.json").read().strip().splitlines()[-1])
                s = d["roofline"]["split"]
                ms.append(f'{d["ms_per_step"]:.2f}(b{s["build_ms"]:.1f}/e{s["eval_ms"]:.1f})')
            except Exception as e:
                ms.append("ERR")
        row.append(f"{c} {ms}")
    print("  ".join(map(str, row)))
PY
tail -2 $O/pytest.txt >> $O/summary.txt
cat $O/summary.txt
