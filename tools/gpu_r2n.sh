#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_resident.py tests/test_gpu_layout.py -m gpu -q -x > $O/r2n_tests.log 2>&1; echo rc=$? >> $O/r2n_tests.log
for v in "VBD_RES_CL=16" "VBD_RESIDENT=0"; do
  echo "== $v" >> $O/r2n_c1.log
  env $v timeout 120 python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --no-fp64-record --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> $O/r2n_c1.log
done
timeout 300 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize.py k1r > $O/r2n_race_k1r.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/sanitize.py k1r > $O/r2n_mem_k1r.log 2>&1
