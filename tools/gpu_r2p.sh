#!/bin/bash
# K1R back on barrier.cluster with push masks; sanitizers over every step kernel
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_resident.py tests/test_gpu_layout.py -m gpu -q -x > $O/r2p_tests.log 2>&1; echo rc=$? >> $O/r2p_tests.log
for v in "VBD_RES_CL=16" "VBD_RESIDENT=0"; do
  echo "== $v" >> $O/r2p_c1.log
  env $v timeout 60 python bench.py --config c1 --steps 100 --warmup 10 --no-cpu-baseline --no-fp64-record --e2e-steps 1 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> $O/r2p_c1.log
done
for t in racecheck memcheck synccheck; do
  for c in k1t k1r k1r_glob k1 explicit fp64 p2p; do
    timeout 300 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py $c > $O/r2p_san_${t}_${c}.log 2>&1
    echo "$t $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $O/r2p_san_${t}_${c}.log | tail -n 2 | tr '\n' ' ')" >> $O/r2p_san_summary.log
  done
done
