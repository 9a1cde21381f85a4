#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for a in 1.0 1.5 1.8 2.0 2.2; do
for c in c1 c2; do
PF_MG_CORR=$a timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mgc_${c}_$a.log 2>&1
grep '^{' gpurun_out/mgc_${c}_$a.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c $a', round(d['value'],3), round(d['ms_per_step'],2), d['iterations_per_step'])" || tail -3 gpurun_out/mgc_${c}_$a.log
done; done
