#!/bin/bash
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_tiles|k2_step|k3_cheb|k4_commit" -c 170 --csv --log-file $O/r5u_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record --e2e-steps 1 > $O/r5u_launches_c5.log 2>&1
