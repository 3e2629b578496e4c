#!/bin/bash
O=gpurun_out
for cfg in "VBD_TILE_OCC=2" "VBD_TILE_OCC=3"; do
  echo "== $cfg" >> $O/r6m.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r6m.log
done
