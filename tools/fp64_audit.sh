#!/bin/bash
# fp64 instruction counts of K1 / K2 per launch (ncu, thread-level dadd/dmul/dfma) for the
# audit against the (2.75-3.25)·L·log2 L model; config c, t columns
mkdir -p gpurun_out/r2
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,launch__grid_size
for spec in "2 0" "5 256"; do
  set -- $spec
  timeout 300 python tools/run_step.py --config $1 --t $2 --steps 1 > gpurun_out/r2/audit_plain_c$1.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_rows16|k_cols|k_pack" --csv \
     python tools/run_step.py --config $1 --t $2 --steps 1 > gpurun_out/r2/fp64_audit_c$1.csv 2>&1
  echo "audit c$1 rc=$?"
done
