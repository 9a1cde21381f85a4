#!/bin/bash
# GPU-box check: gpu tests, smoke, benches (run via gpurun)
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
echo "exit $?" >> gpurun_out/bench_c5.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1
echo "exit $?" >> gpurun_out/bench_c4.log
tail -3 gpurun_out/*.log
