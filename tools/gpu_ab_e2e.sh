# A/B of library variants: parity tests on the default library, C4/C3/C5 evaluation times and the
# C4 host drop-in (e2e) time per variant.   usage: bash tools/gpu_ab_e2e.sh TAG NAME1 NAME2 ...
T=$1; shift
O=gpurun_out/$T
mkdir -p $O
bash tools/gpu_ab_parity.sh $T "$@" > /dev/null 2>&1
for v in "$@"; do
  PF_LIB_PATH=variants/$v.so timeout 600 python tools/e2e_probe.py C4 16 > $O/${v}_e2e.txt 2>&1
  echo "$v $(grep 'ms per call' $O/${v}_e2e.txt)" >> $O/summary.txt
done
cat $O/summary.txt
