#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r5m_tests.log 2>&1
for c in c2 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/r5m_bench_$c.log 2>&1
done
