#!/bin/bash
O=gpurun_out
for tool in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py k1t_class > $O/r5j_san_${tool}.log 2>&1
  echo "$tool rc=$?" >> $O/r5j.log
  grep -E "SUMMARY|hazard" $O/r5j_san_${tool}.log | tail -2 >> $O/r5j.log
done
