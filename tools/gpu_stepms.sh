#!/bin/bash
# repeated default benches with per-step device / host times
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stepms_$rep.log 2>&1
  grep '^{' gpurun_out/stepms_$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print('$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])
print('  dev ', s['device']); print('  host', s['host_issue'])"
done
