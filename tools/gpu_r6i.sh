#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r6i_tests.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r6i_smoke.log 2>&1; echo rc=$? >> $O/r6i_smoke.log
timeout 900 python bench.py > $O/r6i_bench.log 2>&1
timeout 600 python bench.py --config c1 > $O/r6i_bench_c1.log 2>&1
