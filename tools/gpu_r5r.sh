#!/bin/bash
O=gpurun_out
for cfg in "VBD_TILE_CLASS=0 VBD_ENTRY_ORDER=hash" "VBD_TILE_CLASS=0 VBD_ENTRY_ORDER=code" "VBD_TILE_CLASS=1" "VBD_TILE_CLASS=0 VBD_ENTRY_ORDER=hash"; do
  echo "== $cfg" >> $O/r5r.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r5r.log
done
