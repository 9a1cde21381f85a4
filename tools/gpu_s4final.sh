#!/bin/bash
# final measurements of session 4: gpu tier, smoke, same-box Jacobi / Neumann-2 A/B,
# C4 / C5 / C1 bench lines, the C4 step's launch list
mkdir -p gpurun_out/final; cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/final/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -n 1 gpurun_out/final/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/final/smoke.log 2>&1
echo "smoke exit $?"; tail -n 1 gpurun_out/final/smoke.log
for rep in 1 2; do
for mode in jacobi neumann2; do
  PF_MOMENTUM_PRECOND=$mode timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/ab_$mode$rep.log 2>&1
  grep '^{' gpurun_out/final/ab_$mode$rep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode$rep', round(d['value'],1), 'Mcell-steps/s', round(d['ms_per_step'],2), 'ms/step e2e', round(d['e2e']['value'],1), 'sm_mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'], d['iterations_per_step'], 'whole-step kB/cell', d['roofline']['whole_step']['bytes_per_cell']/1e3)" | tee -a gpurun_out/final/r2_nm_light.txt
done
done
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final/bench_c4.log 2>&1
grep '^{' gpurun_out/final/bench_c4.log > gpurun_out/final/r2_bench_c4.json; python -c "
import json; d=json.load(open('gpurun_out/final/r2_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'], d['cpu_baseline']['value'], d['gpu_launches'])"
for c in c5 c1; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final/bench_$c.log 2>&1
grep '^{' gpurun_out/final/bench_$c.log > gpurun_out/final/r2_bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/final/r2_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'])"
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/r2_step_launches_c4_nm.csv python tools/dev/step_launches.py > gpurun_out/final/step.log 2>&1
python tools/launch_summary.py gpurun_out/final/r2_step_launches_c4_nm.csv > gpurun_out/final/r2_step_launches_c4_nm.md 2>&1; tail -1 gpurun_out/final/r2_step_launches_c4_nm.md
