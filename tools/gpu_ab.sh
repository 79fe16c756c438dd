# A/B timing of library variants (variants/NAME.so, tools/build_variant.sh):
# C4 and C3 evaluation times per variant, alternating order twice.
# usage: bash tools/gpu_ab.sh TAG NAME1 NAME2 ...
T=$1; shift
O=gpurun_out/$T
mkdir -p $O
for rep in 1 2; do
  for v in "$@"; do
    for c in C4 C3; do
      PF_LIB_PATH=variants/$v.so timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-newton --no-hbm \
        > $O/${v}_${c}_$rep.json 2> $O/${v}_${c}_$rep.err
    done
  done
done
O=$O python - "$@" <<'PY' > $O/ab_summary.txt
import json, os, sys
O = os.environ["O"]
for v in sys.argv[1:]:
    row = [v]
    for c in ("C4", "C3"):
        ms = []
        for rep in (1, 2):
            try:
                d = json.loads(open(f"{O}/{v}_{c}_{rep}.json").read().strip().splitlines()[-1])
                ms.append(round(d["ms_per_step"], 2))
            except Exception as e:
                ms.append("ERR")
        row.append(f"{c} {ms}")
    print("  ".join(map(str, row)))
PY
cat $O/ab_summary.txt
