#!/bin/bash
mkdir -p gpurun_out/last; cd $GRAFT_REPO_ROOT
for c in c4 c5 c1; do
timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/last/bench_$c.log 2>&1
grep '^{' gpurun_out/last/bench_$c.log > gpurun_out/last/r2_bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/last/r2_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d.get('step_ms',{}).get('e2e_device')[:6])" || tail -5 gpurun_out/last/bench_$c.log
done
