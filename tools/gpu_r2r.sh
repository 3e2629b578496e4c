#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_contacts.py tests/test_gpu_collision.py tests/test_gpu_harness.py tests/test_gpu_energy.py -m gpu -q -x > $O/r2r_tests.log 2>&1; echo rc=$? >> $O/r2r_tests.log
timeout 300 python tools/k1r_slope.py > $O/r2r_slope.log 2>&1
timeout 300 python bench.py --config c5j --scale 0.05 --steps 2 --warmup 3 --no-fp64-record --no-cpu-baseline > $O/r2r_c5j_small.log 2>&1; echo rc=$? >> $O/r2r_c5j_small.log
