#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q > $O/r5q_tests.log 2>&1
for cfg in "VBD_TILE_CLASS_MIX=1" "VBD_TILE_CLASS_MIX=0" "VBD_TILE_CLASS=0" "VBD_TILE_CLASS_MIX=1"; do
  echo "== $cfg" >> $O/r5q.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r5q.log
done
echo "== fp64" >> $O/r5q.log
timeout 300 python tools/k1_once.py c5 fp64 2>&1 | tail -1 >> $O/r5q.log
