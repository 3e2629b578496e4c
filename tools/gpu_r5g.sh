#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r5g_tests.log 2>&1
timeout 900 python bench.py > $O/r5g_bench.log 2>&1
