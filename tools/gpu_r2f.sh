#!/bin/bash
# fp64 split-half position stage: layout/config parity + fp64 C5 timing + ncu of the fp64 K1T
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q > $O/r2f_tests.log 2>&1; echo rc=$? >> $O/r2f_tests.log
timeout 300 python tools/k1_once.py c5 fp64 > $O/r2f_k1_fp64.log 2>&1
timeout 300 python tools/k1_once.py c5 fp32 >> $O/r2f_k1_fp64.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2f_k1t_c5_fp64 python tools/k1_once.py c5 fp64 > $O/r2f_ncu.log 2>&1
