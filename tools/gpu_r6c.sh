#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q -k "class or bitwise" > $O/r6c_tests.log 2>&1
for d in 0 1 0; do
  echo "== VBD_TILE_DBG=$d" >> $O/r6c.log
  VBD_TILE_DBG=$d timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r6c.log
done
echo "== c4" >> $O/r6c.log; timeout 300 python tools/k1_once.py c4 fp32 2>&1 | tail -1 >> $O/r6c.log
echo "== c5 fp64" >> $O/r6c.log; timeout 300 python tools/k1_once.py c5 fp64 2>&1 | tail -1 >> $O/r6c.log
