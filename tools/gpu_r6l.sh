#!/bin/bash
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 8 -c 1 -o $O/r6l_cls_c4 python tools/k1_once.py c4 fp32 > $O/r6l_ncu.log 2>&1
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:k1_ --launch-skip 4 -c 2 --csv --log-file $O/r6l_flops_c4_fp32.csv python tools/k1_once.py c4 fp32 > /dev/null 2>&1
