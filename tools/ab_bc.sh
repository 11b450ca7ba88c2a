#!/bin/bash
# A/B the in-tree library against variant builds under build/<name>, periodic
# (config 4) and walls, in one GPU session: tools/ab_bc.sh name1 name2 ...
for rep in 1 2; do
  for bc in periodic walls; do
    echo "base $bc: $(python tools/prof_stage.py 8192 10 0 x $bc | tail -1)"
    for d in "$@"; do echo "$d $bc: $(HSGN_LIB=build/$d/libhsgn_b200.so python tools/prof_stage.py 8192 10 0 x $bc | tail -1)"; done
  done
done
