#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_layout.py tests/test_gpu_parity.py tests/test_gpu_resident.py -m gpu -q -x > $O/r3u_tests.log 2>&1; echo rc=$? >> $O/r3u_tests.log
for cfg in c2 c3; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3u.log; done
VBD_RESIDENT=0 timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-fp64-record --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | head -1 >> $O/r3u.log
timeout 300 python tools/k1_once.py c5 fp32 2>&1 | tail -1 >> $O/r3u.log
