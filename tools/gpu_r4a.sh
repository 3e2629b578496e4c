#!/bin/bash
O=gpurun_out
for v in 64 32; do
  echo "== fp64 tile_v=$v" >> $O/r4a.log
  VBD_TILE_V=$v timeout 300 python tools/k1_once.py c5 fp64 2>&1 | tail -2 >> $O/r4a.log
  echo "== fp32 tile_v=$v" >> $O/r4a.log
  VBD_TILE_V=$v timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -2 >> $O/r4a.log
done
