#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_resident.py -m gpu -q > $O/r2m_tests.log 2>&1; echo rc=$? >> $O/r2m_tests.log
for v in "VBD_RES_CL=16" "VBD_RES_CL=8" "VBD_RES_CL=16 VBD_RES_PUSH=all" "VBD_RES_CL=8 VBD_RES_PUSH=all" "VBD_RESIDENT=0"; do
  echo "== $v" >> $O/r2m_c1.log
  env $v timeout 120 python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --no-fp64-record --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> $O/r2m_c1.log
done
