#!/bin/bash
# final round-2 bench lines with the class-tile build
O=gpurun_out
timeout 900 python bench.py > $O/r5k_bench_c5.log 2>&1
for c in c4 c3 c2 c1; do
  timeout 900 python bench.py --config $c > $O/r5k_bench_$c.log 2>&1
done
timeout 900 python bench.py --config c5j --no-fp64-record > $O/r5k_bench_c5j.log 2>&1
