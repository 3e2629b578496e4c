#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slab" > $O/r6b_tests.log 2>&1
