#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/cgt.log 2>&1
echo "cgt exit $?" >> gpurun_out/cgt.log
tail -n 4 gpurun_out/cgt.log
for rep in 1 2; do
for mode in tiled gather; do
  if [ $mode = gather ]; then export PF_NO_TILED_CG=1; else unset PF_NO_TILED_CG; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cgt_$mode$rep.log 2>&1
  grep '^{' gpurun_out/cgt_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
cg={n: round(v['ms_per_launch']*1e3,1) for n,v in k.items() if 'cg' in n}
print('$mode$rep', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], cg, d['roofline']['pressure_cg_iteration'])"
done
done
