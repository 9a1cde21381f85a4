#!/bin/bash
# GPU-box: gpu tests + smoke
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
tail -n 30 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log
if [ "$1" == "bench" ]; then
  timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
  timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1
  tail -n 2 gpurun_out/bench_c5.log gpurun_out/bench_c4.log
fi
