#!/bin/bash
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
TAG=${1:-mg}
CFG=${2:-c4}
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 300 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --profile-iters 2 \
  > gpurun_out/ncu_${TAG}.log 2>&1
echo "exit $?" >> gpurun_out/ncu_${TAG}.log
tail -n 2 gpurun_out/ncu_${TAG}.log
