#!/bin/bash
# small-scene bench lines with timed regions long enough for the clock sampler (>= 1 s)
O=gpurun_out
timeout 900 python bench.py --config c1 --steps 10000 --warmup 20 > $O/r6a_bench_c1.log 2>&1
timeout 900 python bench.py --config c2 --steps 600 --warmup 5 > $O/r6a_bench_c2.log 2>&1
timeout 900 python bench.py --config c3 --steps 500 --warmup 5 > $O/r6a_bench_c3.log 2>&1
