#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r5s_tests.log 2>&1
timeout 900 python bench.py > $O/r5s_bench_c5.log 2>&1
timeout 900 python bench.py --config c4 > $O/r5s_bench_c4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 8 -c 1 -o $O/r5s_cls python tools/k1_once.py c5 fp32 > $O/r5s_ncu.log 2>&1
