#!/bin/bash
O=gpurun_out
for cfg in "VBD_TILE_CLASS_HOIST=1" "VBD_TILE_CLASS_HOIST=0"; do
  echo "== $cfg" >> $O/r6h.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -2 >> $O/r6h.log
done
