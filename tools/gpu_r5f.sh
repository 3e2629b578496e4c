#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q -k "class or cover or bitwise" > $O/r5f_tests.log 2>&1
for cfg in "VBD_TILE_CLASS=1" "VBD_TILE_CLASS=0"; do
  echo "== fp32 $cfg" >> $O/r5f.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -3 >> $O/r5f.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 8 -c 1 -o $O/r5f_cls python tools/k1_once.py c5 fp32 > $O/r5f_ncu.log 2>&1
