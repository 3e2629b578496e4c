#!/bin/bash
# class tiles: first GPU check (tests + C5 pass times with / without)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q -k "class or cover or bitwise" > $O/r5a_tests.log 2>&1
for m in 1 0; do
  echo "== fp32 VBD_TILE_CLASS=$m" >> $O/r5a.log
  VBD_TILE_CLASS=$m timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -3 >> $O/r5a.log
done
