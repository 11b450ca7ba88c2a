#!/bin/bash
# ncu counters of the S12 kernel for the in-tree library and variant builds
# under build/<name> (instructions, local-memory traffic, FP64 mix):
#   tools/diag_ab.sh name1 name2 ...
for v in base "$@"; do
  L=""; [ $v != base ] && L="HSGN_LIB=build/$v/libhsgn_b200.so"
  echo "== $v"
  env $L timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none -k "regex:s12" -c 3 --csv python tools/prof_stage.py 8192 4 2>&1 | grep -v "^==" | grep s12_kernel | awk -F'","' '{print $13, $15}'
done
