#!/bin/bash
# stall diagnosis: clock sampler on / slow / off
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
for mode in on off slow; do
  unset PF_NO_CLOCK_SAMPLER PF_CLOCK_MS
  [ $mode = off ] && export PF_NO_CLOCK_SAMPLER=1
  [ $mode = slow ] && export PF_CLOCK_MS=1000
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stepms2_$mode$rep.log 2>&1
  grep '^{' gpurun_out/stepms2_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print('$mode$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['samples'], [round(x) for x in s['device']])"
done
done
