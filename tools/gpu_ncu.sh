#!/bin/bash
# GPU-box: ncu launch list of the bench command + full capture of the top kernels
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 4000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv|k_cg_update|k_cg_pupdate" -s 60 -c 3 \
  -o gpurun_out/prof_cg_${TAG} python bench.py --steps 1 --warmup 0 --no-cpu-baseline --profile-iters 2 \
  > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full_${TAG}.log
tail -n 2 gpurun_out/ncu_launch_${TAG}.log gpurun_out/ncu_full_${TAG}.log
ls -la gpurun_out
