#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/nm_profile.py > gpurun_out/pipe_time.log 2>&1; cat gpurun_out/pipe_time.log
timeout 1200 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_slab.py -m gpu -q -x --timeout 600 > gpurun_out/pipe.log 2>&1
echo "pipe exit $?" >> gpurun_out/pipe.log
tail -n 4 gpurun_out/pipe.log
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches_c4.csv python tools/dev/step_launches.py > gpurun_out/step_launches.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pipe_bench$rep.log 2>&1
  grep '^{' gpurun_out/pipe_bench$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
