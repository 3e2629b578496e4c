#!/bin/bash
O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r5v_smoke.log 2>&1; echo rc=$? >> $O/r5v_smoke.log
timeout 1200 python bench.py --gpus 2 --no-fp64-record > $O/r5v_bench_c5_2ranks.log 2>&1
