#!/bin/bash
# time the default library and every variant under paper_2601_05765_b200/variants (dev tool)
# usage: variants.sh [scenes...]   (c4 via prof_cells.py; C3/C5 via prof_psi.py at converged weights)
SC=${@:-c4}
for r in 1 2; do
for lib in paper_2601_05765_b200/libpotflow_b200.so paper_2601_05765_b200/variants/*.so; do
  echo "== $lib"
  for sc in $SC; do
    case $sc in
      c*) PF_LIB_PATH=$PWD/$lib python tools/prof_cells.py $sc 4 | tail -1 ;;
      *) PF_LIB_PATH=$PWD/$lib python tools/prof_psi.py $sc 2 | tail -1 ;;
    esac
  done
done
done
