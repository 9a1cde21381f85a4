#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
bash tools/sanitize.sh
for c in c5 c5train; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?" >> gpurun_out/bench_$c.log
  grep '^{' gpurun_out/bench_$c.log | cut -c1-400
done
