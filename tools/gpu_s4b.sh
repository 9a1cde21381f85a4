#!/bin/bash
# default (Neumann-2) bench with the matching kernel profile + the step's ncu launch list
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4b_bench.log 2>&1
grep '^{' gpurun_out/s4b_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['iterations_per_step'])
r=d['roofline']; print(r['kernel'], r['frac'], r['share_of_step'])
for k,v in r['kernels'].items(): print(' ', k, round(v['ms_per_launch']*1e3,1), v['launches_per_step'], round(v['share_of_step'],3), round(v['frac'],3))
print(r['whole_step'])"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s4_step_launches_c4.csv python tools/dev/step_launches.py > gpurun_out/s4_step.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/s4_step.log
python tools/launch_summary.py gpurun_out/s4_step_launches_c4.csv > gpurun_out/s4_step_launches_c4.md 2>&1; head -40 gpurun_out/s4_step_launches_c4.md
