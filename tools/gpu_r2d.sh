#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_stage_api.py -m gpu -q -s --timeout 300 > gpurun_out/stage.log 2>&1
echo "stage exit $?" >> gpurun_out/stage.log
grep -E "assert|Error|worst|passed|failed" gpurun_out/stage.log | head -30
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches_c4.csv python tools/dev/step_launches.py > gpurun_out/step_launches.log 2>&1
tail -2 gpurun_out/step_launches.log
