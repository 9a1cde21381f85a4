#!/bin/bash
# same-box A/B of the step: Neumann-2 (default) vs Jacobi, twice each
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for mode in nm jac; do
  if [ $mode = jac ]; then export PF_NO_NEUMANN=1; else unset PF_NO_NEUMANN; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$mode$rep.log 2>&1
  grep '^{' gpurun_out/ab_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
done
done
