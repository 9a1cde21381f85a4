#!/bin/bash
# stall diagnosis: no nvidia-smi at all vs default
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2 3 4 5 6; do
for mode in default; do
  unset PF_NO_CLOCK_SAMPLER PF_NO_IDLE_WAIT
  [ $mode = nosmi ] && export PF_NO_CLOCK_SAMPLER=1 PF_NO_IDLE_WAIT=1
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stepms4_$mode$rep.log 2>&1
  grep '^{' gpurun_out/stepms4_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print('$mode r$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), [round(x) for x in s['device']], [round(x) for x in s['e2e_device']])"
done
done
