#!/bin/bash
O=gpurun_out
for i in 1 2; do
  for p in fp32 fp64; do
    echo "== old $p" >> $O/r5t.log; timeout 300 python _old/k1_once_old.py c5 $p 2>&1 | tail -1 >> $O/r5t.log
    echo "== new plain $p" >> $O/r5t.log; VBD_TILE_CLASS=0 timeout 300 python tools/k1_once.py c5 $p 2>&1 | tail -1 >> $O/r5t.log
  done
done
