#!/bin/bash
mkdir -p gpurun_out/final; cd $GRAFT_REPO_ROOT
for c in c1 c5; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final/bench_$c.log 2>&1
grep '^{' gpurun_out/final/bench_$c.log > gpurun_out/final/r2_bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/final/r2_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'], d['iterations_per_step'])"
done
