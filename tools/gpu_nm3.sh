#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/nm_profile.py > gpurun_out/nm_time3.log 2>&1
PF_NM_MINB=1 timeout 300 python tools/dev/nm_profile.py >> gpurun_out/nm_time3.log 2>&1
cat gpurun_out/nm_time3.log
timeout 900 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py -m gpu -q -x --timeout 300 > gpurun_out/nm3.log 2>&1
echo "nm exit $?" >> gpurun_out/nm3.log
tail -n 5 gpurun_out/nm3.log
