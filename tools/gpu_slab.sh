#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
PF_BENCH_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --config slab8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/selflaunch.log 2>&1
echo "selflaunch exit $?" >> gpurun_out/selflaunch.log
grep '^{' gpurun_out/selflaunch.log | cut -c1-250; tail -2 gpurun_out/selflaunch.log
for w in 1 2 8; do
  timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/slab_overhead_$w.log 2>&1
  tail -3 gpurun_out/slab_overhead_$w.log
done
