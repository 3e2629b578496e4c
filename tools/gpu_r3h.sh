#!/bin/bash
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_layout.py -m gpu -q -k "k1t_explicit or jittered" > $O/r3h_tests.log 2>&1; echo rc=$? >> $O/r3h_tests.log
for v in "VBD_TILES_X=1" "VBD_TILES_X=1 VBD_TILE_OCC=3"; do
  echo "== c5j $v" >> $O/r3h.log
  env $v timeout 300 python tools/k1_once.py c5j fp32 2>&1 | tail -1 >> $O/r3h.log
done
