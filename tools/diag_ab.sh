bash tools/ab_bc.sh early steady > gpurun_out/ab_early.txt 2>&1; cat gpurun_out/ab_early.txt
for v in base steady; do
  L=""; [ $v != base ] && L="HSGN_LIB=build/$v/libhsgn_b200.so"
  env $L timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none -k "regex:s12" -c 3 --csv python tools/prof_stage.py 8192 4 > gpurun_out/diag_$v.csv 2>&1
  grep -v "^==" gpurun_out/diag_$v.csv | cut -c1-400 | tail -25
done
