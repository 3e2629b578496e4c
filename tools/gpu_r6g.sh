#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_parity.py -x -q -k "class or bitwise or slab" > $O/r6g_tests.log 2>&1
for cfg in "VBD_TILE_CLASS_HOIST=1" "VBD_TILE_CLASS_HOIST=0" "VBD_TILE_CLASS_HOIST=1"; do
  echo "== $cfg" >> $O/r6g.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r6g.log
done
echo "== c4" >> $O/r6g.log; timeout 300 python tools/k1_once.py c4 fp32 2>&1 | tail -1 >> $O/r6g.log
