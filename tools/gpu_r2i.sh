#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2i.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2i.log
tail -n 3 gpurun_out/r2i.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench.log 2>&1
grep '^{' gpurun_out/r2i_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['roofline']['whole_step']['frac'], d['roofline']['pressure_cg_iteration'])"
bash tools/gpu_ncu_final.sh
