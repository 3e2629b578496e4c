#!/bin/bash
# round-2 GPU call: config parity tests, self-spawned bench test, C5 bench line, FP counters
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_bench.py -x -q -s > $O/r2c_tests.log 2>&1; echo rc=$? >> $O/r2c_tests.log
timeout 600 python bench.py > $O/r2c_bench_c5.log 2>&1
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cp in "c5 fp32" "c5 fp64" "c4 fp32" "c4 fp64"; do
  set -- $cp
  timeout 300 ncu --metrics $M --clock-control none -k regex:k1_ --launch-skip 4 -c 2 --csv --log-file $O/r2c_flops_$1_$2.csv python tools/k1_once.py $1 $2 > /dev/null 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -k regex:k_fma_peak -c 3 --csv --log-file $O/r2c_flops_fma.csv python tools/k1_once.py x x --fma > $O/r2c_fma.log 2>&1
python tools/k1_once.py x x --fma >> $O/r2c_fma.log 2>&1
