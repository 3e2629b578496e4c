#!/bin/bash
O=gpurun_out
for rep in 1 2; do
for e in 1 0; do
  echo "== early=$e" >> $O/r3v.log
  for cfg in c2 c3; do VBD_PDL_EARLY=$e timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3v.log; done
  VBD_PDL_EARLY=$e VBD_RESIDENT=0 timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3v.log
  VBD_PDL_EARLY=$e timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r3v.log
done
done
