#!/bin/bash
# A/B of the adaptive and sourced S12 paths: the in-tree library against
# variant builds under build/<name> (bench.py --adaptive; config-2 rungs)
for rep in 1 2; do
  for v in base "$@"; do
    L=""; [ $v != base ] && L="HSGN_LIB=build/$v/libhsgn_b200.so"
    a=$(env $L timeout 300 python bench.py --adaptive 1e-8 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), round(d['ms_per_step'],3))")
    c=$(env $L timeout 300 python tools/config2_rungs.py 0.02 2048,4096 2>/dev/null | awk '{print $1, $2, $3, $NF, $(NF-2)}' | tr '\n' ' ')
    echo "$v adaptive G/s, ms/attempt: $a | config2 rungs: $c"
  done
done
