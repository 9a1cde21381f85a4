#!/bin/bash
# Neumann-2 as the default: whole gpu tier, smoke, A/B x2, default bench
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
tail -n 2 gpurun_out/smoke.log
for rep in 1 2; do
for mode in jacobi neumann2; do
  PF_MOMENTUM_PRECOND=$mode timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nmdef_$mode$rep.log 2>&1
  grep '^{' gpurun_out/nmdef_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['iterations_per_step'])"
done
done
