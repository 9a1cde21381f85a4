#!/bin/bash
# GPU-box: whole gpu tier, smoke, default C4 bench
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
tail -n 2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c4.log
grep '^{' gpurun_out/bench_c4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['iterations_per_step'])
for k,v in r['kernels'].items(): print(f\"{k:32s} {v['ms_per_launch']*1e3:7.1f}us x{v['launches_per_step']:4.1f} share {v['share_of_step']:.3f} frac {v['frac']:.2f}\")"
