#!/bin/bash
# same-box A/B: speculative solver close vs close-after-poll
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for mode in spec poll; do
  if [ $mode = poll ]; then export PF_NO_SPECULATIVE=1; else unset PF_NO_SPECULATIVE; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/spec_$mode$rep.log 2>&1
  grep '^{' gpurun_out/spec_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['iterations_per_step'])"
done
done
