#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > $O/r5x_tests.log 2>&1
timeout 900 python tools/k1r_slope_c2.py c2 > $O/r5x_slope.log 2>&1
