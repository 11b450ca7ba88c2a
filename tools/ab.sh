#!/bin/bash
# A/B the in-tree library against variant builds under build/<name> in one GPU session.
for rep in 1 2; do
  echo "base: $(python tools/prof_stage.py 8192 10 0 x | tail -1)"
  for d in "$@"; do echo "$d: $(HSGN_LIB=build/$d/libhsgn_b200.so python tools/prof_stage.py 8192 10 0 x | tail -1)"; done
done
