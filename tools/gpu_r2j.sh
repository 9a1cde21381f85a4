#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_slab_ipc.py -m gpu -q --timeout 600 > gpurun_out/r2j_new.log 2>&1
echo "new exit $?" >> gpurun_out/r2j_new.log; tail -n 4 gpurun_out/r2j_new.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches_c4_final.csv python tools/dev/step_launches.py > gpurun_out/step_final.log 2>&1
tail -1 gpurun_out/step_final.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench$rep.log 2>&1
  grep '^{' gpurun_out/r2j_bench$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['roofline']['whole_step']['frac'], d.get('other_gpu_processes'))"
done
