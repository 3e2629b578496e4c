#!/bin/bash
# after the displacement state + K1R: whole GPU suite (prints kept), bench C5 / C1, ncu of fp32 K1T
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -s > $O/r2l_all.log 2>&1; echo rc=$? >> $O/r2l_all.log
timeout 600 python bench.py > $O/r2l_bench_c5.log 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-fp64-record > $O/r2l_bench_c1.log 2>&1
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-fp64-record > $O/r2l_bench_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2l_k1t_c5_fp32 python tools/k1_once.py c5 fp32 > $O/r2l_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_step_resident -c 1 -o $O/r2l_k1r_c1 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record > $O/r2l_ncu_c1.log 2>&1
