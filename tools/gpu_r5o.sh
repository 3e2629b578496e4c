#!/bin/bash
O=gpurun_out
for d in 0 1 2; do
  echo "== VBD_TILE_DBG=$d" >> $O/r5o.log
  VBD_TILE_DBG=$d timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r5o.log
done
