#!/bin/bash
# class tiles: FP counters + DRAM bytes (C5, C4 fp32), C4 bench line, C5 launch list
O=gpurun_out
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in c5 c4; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k1_ --launch-skip 4 -c 2 --csv --log-file $O/r5h_flops_${c}_fp32.csv python tools/k1_once.py $c fp32 > $O/r5h_once_$c.log 2>&1
done
timeout 900 python bench.py --config c4 --no-fp64-record > $O/r5h_bench_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r5h_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record > /dev/null 2>&1
