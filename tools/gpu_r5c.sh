#!/bin/bash
O=gpurun_out
for cfg in "VBD_TILE_CLASS=0 VBD_ENTRY_ORDER=hash" "VBD_TILE_CLASS=0" "VBD_TILE_CLASS=1" "VBD_TILE_CLASS=0 VBD_ENTRY_ORDER=hash"; do
  echo "== fp32 $cfg" >> $O/r5c.log
  env $cfg timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -3 >> $O/r5c.log
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv >> $O/r5c.log
