#!/bin/bash
for t in 4 8 16; do
  echo "== threads $t" >> gpurun_out/r3s.log
  VBD_STAGE_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --no-fp64-record --steps 3 --warmup 3 --e2e-steps 2 2>&1 | grep -o '"e2e": {[^}]*}[^}]*}' >> gpurun_out/r3s.log
done
nproc >> gpurun_out/r3s.log
