#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/r3i_all.log 2>&1; echo rc=$? >> $O/r3i_all.log
timeout 900 python bench.py --config c5j --steps 3 --warmup 3 --no-fp64-record > $O/r3i_bench_c5j.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r3i_k1tx_c5j python tools/k1_once.py c5j fp32 > $O/r3i_ncu.log 2>&1
