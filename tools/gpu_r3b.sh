#!/bin/bash
O=gpurun_out
for v in "VBD_K1=4x2b3" "VBD_K1=8x1" "VBD_K1=4x1" "VBD_K1=4x2b3p1"; do
  echo "== c5j $v" >> $O/r3b.log
  env $v timeout 200 python tools/k1_once.py c5j fp32 2>&1 | tail -1 >> $O/r3b.log
done
