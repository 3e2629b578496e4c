#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_layout.py tests/test_gpu_resident.py tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > $O/r3e_tests.log 2>&1; echo rc=$? >> $O/r3e_tests.log
for v in "VBD_TILES_X=1" "VBD_TILES_X=0"; do
  echo "== c5j $v" >> $O/r3e.log
  env $v timeout 300 python tools/k1_once.py c5j fp32 2>&1 | tail -2 >> $O/r3e.log
done
