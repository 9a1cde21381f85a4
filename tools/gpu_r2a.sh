#!/bin/bash
# GPU-box: new live-reference parity tests first, then the whole gpu tier,
# smoke, and one default bench run
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ref_live.py -m gpu -q -s --timeout 600 > gpurun_out/ref_live.log 2>&1
echo "ref_live exit $?" >> gpurun_out/ref_live.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c4.log
tail -n 25 gpurun_out/ref_live.log; tail -n 5 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench_c4.log
