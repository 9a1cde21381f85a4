#!/bin/bash
# GPU-box: per-kernel launch list of ONE fwd+adjoint step (cold-cache,
# serialised by ncu) + plain timing of the same step
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
CFG=${1:-c4}
TAG=${2:-r1}
timeout 600 python tools/step_profile.py --config $CFG > gpurun_out/step_${CFG}_${TAG}.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CFG}_${TAG}.csv python tools/step_profile.py --config $CFG \
  >> gpurun_out/step_${CFG}_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/step_${CFG}_${TAG}.log
python tools/launch_summary.py gpurun_out/launches_${CFG}_${TAG}.csv > gpurun_out/launches_${CFG}_${TAG}.md
cat gpurun_out/step_${CFG}_${TAG}.log; head -n 40 gpurun_out/launches_${CFG}_${TAG}.md
