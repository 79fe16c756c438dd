#!/bin/bash
# Build a variant of the CUDA library into variants/NAME.so (dev tool for A/B
# timing on the GPU box: PF_LIB_PATH=variants/NAME.so python bench.py ...).
# usage: tools/build_variant.sh NAME [GIT_REF|-] [extra nvcc flags...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; REF=${2:--}; shift; shift || true
OUT=$ROOT/variants/$NAME.so
mkdir -p $ROOT/variants
if [ "$REF" = "-" ]; then
  SRC=$ROOT
else
  SRC=/tmp/pf_wt_$NAME
  rm -rf $SRC; git -C $ROOT worktree prune
  git -C $ROOT worktree add -f --detach $SRC $REF >/dev/null 2>&1
fi
# own object directory; extra flags (e.g. -DPF_X=1, EVAL_FMAD=true) through the Makefile
MK=(); EX=()
for a in "$@"; do case "$a" in *=*) if [[ "$a" == -* ]]; then EX+=("$a"); else MK+=("$a"); fi;; *) EX+=("$a");; esac; done
make -s -j6 -C $SRC/paper_2601_05765_b200/csrc OBJDIR=/tmp/pf_obj_$NAME PTXAS_OUT=/tmp/ptxas_$NAME OUT=$OUT \
    EXTRA="${EX[*]}" "${MK[@]}" > /tmp/make_$NAME.log 2>&1 || { tail -20 /tmp/make_$NAME.log; exit 1; }
rm -rf /tmp/pf_obj_$NAME
if [ "$REF" != "-" ]; then git -C $ROOT worktree remove --force $SRC; fi
echo built $OUT
