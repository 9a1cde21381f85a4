#!/bin/bash
# session re-entry check: whole gpu tier, smoke, default bench + Jacobi A/B
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
tail -n 2 gpurun_out/smoke.log
for mode in default jacobi; do
  if [ $mode == default ]; then unset PF_MOMENTUM_PRECOND; else export PF_MOMENTUM_PRECOND=$mode; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4a_$mode.log 2>&1
  grep '^{' gpurun_out/s4a_$mode.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['iterations_per_step'], d['roofline']['name'], d['roofline']['frac'])"
done
