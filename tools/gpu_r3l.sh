#!/bin/bash
# round-2 final record: whole GPU suite, smoke, bench lines C1..C5 + C5j, 2-rank self-spawned C5 (one GPU)
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/r3l_all.log 2>&1; echo rc=$? >> $O/r3l_all.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/r3l_smoke.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r3l_bench_c5.log 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-fp64-record > $O/r3l_bench_c1.log 2>&1
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-fp64-record --no-cpu-baseline > $O/r3l_bench_c2.log 2>&1
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-fp64-record > $O/r3l_bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $O/r3l_bench_c4.log 2>&1
timeout 900 python bench.py --config c5j --steps 3 --warmup 3 --no-fp64-record > $O/r3l_bench_c5j.log 2>&1
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-fp64-record --no-cpu-baseline > $O/r3l_bench_c5_2ranks.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/r3l_bench_ref.log 2>&1
