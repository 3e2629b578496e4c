#!/bin/bash
# final validation of the round's last build: GPU suite, smoke, the driver's default bench, reference arm
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r6d_tests.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r6d_smoke.log 2>&1; echo rc=$? >> $O/r6d_smoke.log
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > $O/r6d_bench.log 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 > $O/r6d_bench_ref.log 2>&1
