#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_tiles|k2_step|k3_cheb|k4_commit" -c 170 --csv --log-file $O/r2y_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp64-record --e2e-steps 1 > $O/r2y_launches_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2y_k1t_c5_fp32 python tools/k1_once.py c5 fp32 > $O/r2y_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tiles --launch-skip 4 -c 1 -o $O/r2y_k1t_c5_fp64 python tools/k1_once.py c5 fp64 > $O/r2y_ncu2.log 2>&1
du -sh $O
