#!/bin/bash
# same-box A/B: Jacobi vs Neumann-2 momentum preconditioner, with kernel tables
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for mode in jac nm; do
  if [ $mode = nm ]; then export PF_MOMENTUM_PRECOND=neumann2; else unset PF_MOMENTUM_PRECOND; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nmab_$mode.log 2>&1
  grep '^{' gpurun_out/nmab_$mode.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$mode', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['iterations_per_step'], d['clocks']['sm_mhz'])
tot=0
for k,v in r['kernels'].items():
  tot+=v['share_of_step']
  print(f\"{k:32s} {v['ms_per_launch']*1e3:7.1f}us x{v['launches_per_step']:4.1f} share {v['share_of_step']:.3f} frac {v['frac']:.2f}\")
print('sum share', round(tot,3))"
done
