#!/bin/bash
# K1R resident step kernel: bitwise tests + small-scene timings (graph vs cluster vs grid)
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_resident.py -m gpu -q -x > $O/r2g_tests.log 2>&1; echo rc=$? >> $O/r2g_tests.log
for cfg in c1 c2 c3; do
  for mode in 0 repl glob; do
    VBD_RESIDENT=$mode timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-fp64-record --e2e-steps 2 > $O/r2g_bench_${cfg}_${mode}.log 2>&1
  done
done
timeout 900 python -m pytest tests -m gpu -q > $O/r2g_all.log 2>&1; echo rc=$? >> $O/r2g_all.log
