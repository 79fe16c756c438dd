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
make -s -C $SRC/paper_2601_05765_b200/csrc -B OUT=$OUT NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xptxas -v $*" > /tmp/ptxas_$NAME.log 2>&1 || { cat /tmp/ptxas_$NAME.log | tail -20; exit 1; }
if [ "$REF" != "-" ]; then git -C $ROOT worktree remove --force $SRC; fi
echo built $OUT
