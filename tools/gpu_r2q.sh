#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_layout.py tests/test_gpu_resident.py tests/test_gpu_parity.py -m gpu -q > $O/r2q_tests.log 2>&1; echo rc=$? >> $O/r2q_tests.log
timeout 900 python bench.py --config c5j --steps 3 --warmup 3 --no-fp64-record > $O/r2q_bench_c5j.log 2>&1
for t in racecheck memcheck; do
  timeout 300 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py slabs > $O/r2q_san_${t}_slabs.log 2>&1
  echo "$t slabs rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/r2q_san_${t}_slabs.log | tail -n 1)" >> $O/r2q_san_summary.log
done
