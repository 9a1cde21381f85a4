#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_configs.py tests/test_gpu_slab.py -m gpu -q -x --timeout 600 > gpurun_out/cgt2.log 2>&1
echo "cgt exit $?" >> gpurun_out/cgt2.log
tail -n 3 gpurun_out/cgt2.log
for mode in tiled gather; do
  if [ $mode = gather ]; then export PF_NO_TILED_CG=1; else unset PF_NO_TILED_CG; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cgt2_$mode.log 2>&1
  grep '^{' gpurun_out/cgt2_$mode.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
cg={n: round(v['ms_per_launch']*1e3,1) for n,v in k.items() if 'cg' in n}
print('$mode', round(d['value'],1), round(d['ms_per_step'],2), cg, d['roofline']['pressure_cg_iteration'])"
done
