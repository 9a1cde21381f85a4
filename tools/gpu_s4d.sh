#!/bin/bash
# whole gpu tier + smoke, default bench x2, the step's launch list, ysolve ncu
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -n 1 gpurun_out/smoke.log
for rep in 1 2; do
  timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/s4d_bench$rep.log 2>&1
  grep '^{' gpurun_out/s4d_bench$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks'], d['iterations_per_step'], d['cpu_baseline']['value'])
r=d['roofline']
for k,v in r['kernels'].items(): print(' ', k, round(v['ms_per_launch']*1e3,1), round(v['frac'],3))"
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s4d_step_launches_c4.csv python tools/dev/step_launches.py > gpurun_out/s4d_step.log 2>&1
python tools/launch_summary.py gpurun_out/s4d_step_launches_c4.csv > gpurun_out/s4d_step_launches_c4.md 2>&1; head -16 gpurun_out/s4d_step_launches_c4.md
mkdir -p gpurun_out/ncu_nm
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_spec_ysolve --launch-count 1 -o /tmp/ys -f python tools/dev/step_launches.py > gpurun_out/ncu_nm/ys.log 2>&1
ncu -i /tmp/ys.ncu-rep --page details --csv > gpurun_out/ncu_nm/05_k_spec_ysolve.csv 2>/dev/null
ncu -i /tmp/ys.ncu-rep --page raw --csv > gpurun_out/ncu_nm/05_k_spec_ysolve_raw.csv 2>/dev/null
