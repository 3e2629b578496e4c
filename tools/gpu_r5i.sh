#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q -k "class or cover or bitwise" > $O/r5i_tests.log 2>&1
for c in c4 c5; do
  echo "== $c" >> $O/r5i.log
  timeout 300 python tools/k1_once.py $c fp32 2>&1 | tail -2 >> $O/r5i.log
done
