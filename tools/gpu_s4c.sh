#!/bin/bash
# compact q1 ring: Neumann-2 tests, then 1 vs 2 CTAs per SM
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py -m gpu -q --timeout 600 -x > gpurun_out/s4c_test.log 2>&1
echo "pytest exit $?"; tail -n 3 gpurun_out/s4c_test.log
for mb in 1 2 1 2; do
  PF_NM_MINB=$mb timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4c_mb$mb.log 2>&1
  grep '^{' gpurun_out/s4c_mb$mb.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('minb $mb', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['iterations_per_step'])
r=d['roofline']
for k,v in r['kernels'].items():
  if 'nm' in k: print(' ', k, round(v['ms_per_launch']*1e3,1), round(v['frac'],3))"
done
