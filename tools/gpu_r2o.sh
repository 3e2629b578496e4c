#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 200 python -m pytest tests/test_gpu_resident.py -m gpu -q -x > $O/r2o_tests.log 2>&1; echo rc=$? >> $O/r2o_tests.log
for v in "VBD_RES_CL=16" "VBD_RESIDENT=0"; do
  echo "== $v" >> $O/r2o_c1.log
  env $v timeout 60 python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --no-fp64-record --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> $O/r2o_c1.log
done
