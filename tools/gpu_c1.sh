#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1_bench.log 2>&1
grep '^{' gpurun_out/c1_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['ms_per_step'],2), d.get('step_ms'), d['gpu_launches'], d['iterations_per_step'])"
bash tools/gpu_step_ncu.sh c1 s4 > /dev/null 2>&1
head -30 gpurun_out/launches_c1_s4.md; tail -3 gpurun_out/launches_c1_s4.md
