#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
for pp in auto jacobi auto jacobi; do
PF_PRESSURE_PRECOND=$pp timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1_$pp.log 2>&1
grep '^{' gpurun_out/c1_$pp.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$pp', round(d['value'],3), round(d['ms_per_step'],2), d['gpu_launches'], d['iterations_per_step'])"
done
for c in c2 c5; do
for pp in auto jacobi; do
PF_PRESSURE_PRECOND=$pp timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${c}_$pp.log 2>&1
grep '^{' gpurun_out/${c}_$pp.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c $pp', round(d['value'],3), round(d['ms_per_step'],2), d['gpu_launches'], d['iterations_per_step'])"
done; done
