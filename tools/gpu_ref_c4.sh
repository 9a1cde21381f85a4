#!/bin/bash
# GPU-box host: the reference arm on the SAME C4 config (one full taped
# fwd + FULL adjoint step on one core); result -> gpurun_out/ref_c4.json
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/ref_c4_host.txt; lscpu | head -20 >> gpurun_out/ref_c4_host.txt; free -g >> gpurun_out/ref_c4_host.txt
PF_REF_BUDGET_S=2700 timeout 2800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c4.log 2> gpurun_out/ref_c4.err
echo "exit $?" >> gpurun_out/ref_c4.log
grep '^{' gpurun_out/ref_c4.log | tail -1 > gpurun_out/ref_c4.json
tail -c 1500 gpurun_out/ref_c4.log; tail -5 gpurun_out/ref_c4.err
