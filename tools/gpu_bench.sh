#!/bin/bash
# GPU-box: benches (run via gpurun)
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
echo "exit $?" >> gpurun_out/bench_c5.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1
echo "exit $?" >> gpurun_out/bench_c4.log
for f in gpurun_out/bench_c5.log gpurun_out/bench_c4.log; do tail -n 3 $f; done
