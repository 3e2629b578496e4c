#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_bench.py -q -s > $O/r2d_tests.log 2>&1; echo rc=$? >> $O/r2d_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/r2d_bench_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2d_k1t_c5_fp32 python tools/k1_once.py c5 fp32 > $O/r2d_ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2d_k1t_c5_fp64 python tools/k1_once.py c5 fp64 > $O/r2d_ncu2.log 2>&1
ls -la $O/*.ncu-rep
