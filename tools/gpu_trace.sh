#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
rm -f gpurun_out/trace_*.json
for rep in 1 2 3 4 5 6; do
  PF_TRACE_STEPS=1 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/trace_b$rep.log 2>&1
  grep '^{' gpurun_out/trace_b$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print('r$rep', round(d['ms_per_step'],2), [round(x) for x in s['device']])"
done
python tools/dev/trace.py gpurun_out/trace_*.json > gpurun_out/trace_summary.txt
