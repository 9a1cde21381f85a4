#!/bin/bash
mkdir -p gpurun_out/last; cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/last/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/last/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/last/smoke.log 2>&1
echo "smoke exit $?"; tail -n 1 gpurun_out/last/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/last/bench_c4.log 2>&1
grep '^{' gpurun_out/last/bench_c4.log > gpurun_out/last/r2_bench_c4.json; python -c "
import json; d=json.load(open('gpurun_out/last/r2_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])"
