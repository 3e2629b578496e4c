#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q -k "class" > $O/r6f_tests.log 2>&1
timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r6f.log
