#!/bin/bash
O=gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-fp64-record > $O/r6j_bench.log 2>&1
