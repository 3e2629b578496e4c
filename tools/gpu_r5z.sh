#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r5z_tests.log 2>&1
for c in c2 c1 c3; do
  timeout 900 python bench.py --config $c > $O/r5z_bench_$c.log 2>&1
done
