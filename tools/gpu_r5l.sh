#!/bin/bash
O=gpurun_out
for c in c2 c3; do
  for e in code hash code hash; do
    echo "== $c $e" >> $O/r5l.log
    VBD_ENTRY_ORDER=$e timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config'].get('layout')[:60])" >> $O/r5l.log
  done
done
