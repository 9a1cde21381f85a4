#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/nm_profile.py > gpurun_out/jm_time.log 2>&1
PF_NO_MERGE=1 timeout 300 python tools/dev/nm_profile.py >> gpurun_out/jm_time.log 2>&1
cat gpurun_out/jm_time.log
timeout 1200 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_configs.py -m gpu -q -x --timeout 600 > gpurun_out/jm.log 2>&1
echo "jm exit $?" >> gpurun_out/jm.log
tail -n 8 gpurun_out/jm.log
