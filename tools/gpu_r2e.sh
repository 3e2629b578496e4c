#!/bin/bash
# round-2 GPU call: whole GPU suite, smoke, default bench line, ncu full captures of K1T fp32/fp64 C5
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r2e_tests.log 2>&1; echo rc=$? >> $O/r2e_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2e_smoke.log 2>&1
timeout 600 python bench.py > $O/r2e_bench_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2e_k1t_c5_fp32 python tools/k1_once.py c5 fp32 > $O/r2e_ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2e_k1t_c5_fp64 python tools/k1_once.py c5 fp64 > $O/r2e_ncu2.log 2>&1
ls -la $O/
