#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_resident.py -x -q > $O/r5n_tests.log 2>&1
for i in 1 2; do timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r5n.log; done
