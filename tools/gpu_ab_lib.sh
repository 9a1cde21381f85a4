#!/bin/bash
# same-box A/B of two library builds (libpisob200_a.so / _b.so), alternating
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
L=paper_2505_16992_b200
for v in a b a b; do
  cp $L/libpisob200_$v.so $L/libpisob200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  grep '^{' gpurun_out/ab_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['iterations_per_step'])
r=d['roofline']
for k,v in list(r['kernels'].items())[:6]: print(' ', k, round(v['ms_per_launch']*1e3,1), round(v['frac'],3))"
done
