#!/bin/bash
O=gpurun_out
for v in "VBD_TILE_OCC=" "VBD_TILE_OCC=3"; do
  echo "== fp64 $v" >> $O/r3c.log
  env $v timeout 200 python tools/k1_once.py c5 fp64 2>&1 | tail -2 >> $O/r3c.log
done
echo "== fp32" >> $O/r3c.log
timeout 200 python tools/k1_once.py c5 fp32 2>&1 | tail -2 >> $O/r3c.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/r3c_ref.log 2>&1
