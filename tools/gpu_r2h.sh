#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/nm_profile.py > gpurun_out/nm_time4.log 2>&1; cat gpurun_out/nm_time4.log
timeout 1200 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_ref_live.py -m gpu -q -x --timeout 600 > gpurun_out/nm4.log 2>&1
echo "nm exit $?" >> gpurun_out/nm4.log
tail -n 15 gpurun_out/nm4.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
grep '^{' gpurun_out/bench_c4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['iterations_per_step'], r['whole_step'])
for k,v in r['kernels'].items(): print(f\"{k:32s} {v['ms_per_launch']*1e3:7.1f}us x{v['launches_per_step']:4.1f} share {v['share_of_step']:.3f} frac {v['frac']:.2f}\")"
tail -3 gpurun_out/bench_c4.log | cut -c1-300
