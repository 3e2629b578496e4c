#!/bin/bash
O=gpurun_out
for v in "VBD_TILE_W=2" "VBD_TILE_W=4" "VBD_TILE_W=4 VBD_TILE_STAGES=2" "VBD_TILE_W=2 VBD_TILE_OCC=2"; do
  echo "== fp64 $v" >> $O/r2z.log
  env $v timeout 200 python tools/k1_once.py c5 fp64 2>&1 | tail -1 >> $O/r2z.log
done
for v in "VBD_TILE_W=2" "VBD_TILE_W=4"; do
  echo "== fp32 $v" >> $O/r2z.log
  env $v timeout 200 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r2z.log
done
