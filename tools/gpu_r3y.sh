#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_parity.py tests/test_gpu_resident.py tests/test_gpu_configs.py -m gpu -q -x > $O/r3y_tests.log 2>&1; echo rc=$? >> $O/r3y_tests.log
for rep in 1 2; do
for v in 32 64; do
  echo "== tile_v=$v" >> $O/r3y.log
  for cfg in c2 c3; do VBD_TILE_V=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3y.log; done
  VBD_TILE_V=$v VBD_RESIDENT=0 timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3y.log
done
done
