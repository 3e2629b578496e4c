#!/bin/bash
O=gpurun_out
for d in 0 0; do
  echo "== VBD_TILE_DBG=$d" >> $O/r5w.log
  VBD_TILE_DBG=$d timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r5w.log
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv >> $O/r5w.log
