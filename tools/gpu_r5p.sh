#!/bin/bash
# final round-2 bench lines (class-tile build)
O=gpurun_out
timeout 900 python bench.py > $O/r5p_bench_c5.log 2>&1
for c in c4 c3 c2 c1; do
  timeout 900 python bench.py --config $c > $O/r5p_bench_$c.log 2>&1
done
timeout 900 python bench.py --config c5j --no-fp64-record > $O/r5p_bench_c5j.log 2>&1
timeout 900 python bench.py --impl reference > $O/r5p_bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r5p_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record > /dev/null 2>&1
