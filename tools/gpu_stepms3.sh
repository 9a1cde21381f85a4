#!/bin/bash
# stall diagnosis: warmup 3 vs 12
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
for w in 3 12; do
  timeout 600 python bench.py --steps 10 --warmup $w --no-cpu-baseline > gpurun_out/stepms3_$w$rep.log 2>&1
  grep '^{' gpurun_out/stepms3_$w$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print('w$w r$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), [round(x) for x in s['device']], [round(x) for x in s['e2e_device']])"
done
done
nvidia-smi -q -d CLOCK,PERFORMANCE | head -60 > gpurun_out/clockinfo.txt
