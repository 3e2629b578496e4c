#!/bin/bash
O=gpurun_out
for c in c2 c3; do
  for m in glob 0 glob 0; do
    echo "== $c VBD_RESIDENT=$m" >> $O/r5y.log
    VBD_RESIDENT=$m timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['gpu_launches'], d['roofline'].get('step_kernel','graph')[:40])" >> $O/r5y.log
  done
done
