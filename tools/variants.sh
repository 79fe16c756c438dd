#!/bin/bash
# time the default library and every variant under paper_2601_05765_b200/variants (dev tool)
for r in 1 2; do
for lib in paper_2601_05765_b200/libpotflow_b200.so paper_2601_05765_b200/variants/*.so; do
  echo "== $lib"
  for sc in c4; do PF_LIB_PATH=$PWD/$lib python tools/prof_cells.py $sc 4 | tail -1; done
done
done
