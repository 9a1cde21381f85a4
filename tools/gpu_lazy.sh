#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_slab.py -q -x --timeout 600 > gpurun_out/lazy_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/lazy_tests.log; tail -2 gpurun_out/lazy_tests.log
bash tools/gpu_trace.sh
grep -E "^step 2|allocator" gpurun_out/trace_summary.txt | head -12
