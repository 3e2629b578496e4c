#!/bin/bash
# round-2 record (logs only): whole GPU suite, smoke, bench lines C1..C5 + C5j, ncu launch list of the C5 step
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/r2w_all.log 2>&1; echo rc=$? >> $O/r2w_all.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2w_smoke.log 2>&1
timeout 600 python bench.py > $O/r2w_bench_c5.log 2>&1
for cfg in c1 c2 c3; do timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-fp64-record > $O/r2w_bench_$cfg.log 2>&1; done
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $O/r2w_bench_c4.log 2>&1
timeout 900 python bench.py --config c5j --steps 3 --warmup 3 --no-fp64-record > $O/r2w_bench_c5j.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2w_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record --e2e-steps 1 > $O/r2w_launches_c5.log 2>&1
du -sh $O
