#!/bin/bash
O=gpurun_out
for tool in racecheck memcheck synccheck; do
  for c in k1r_glob k1t_class; do
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py $c > $O/r6k_san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'SUMMARY' $O/r6k_san_${tool}_$c.log | tail -1)" >> $O/r6k.log
  done
done
