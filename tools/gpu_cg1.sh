#!/bin/bash
# single-reduction CG: tests, slab tests, slab overhead classic vs single
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_cg_single.py tests/test_gpu_slab.py tests/test_gpu_slab_ipc.py -q -x --timeout 600 -s > gpurun_out/cg1_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/cg1_tests.log
grep -E "single-reduction|passed|failed|Error" gpurun_out/cg1_tests.log | tail -8
for v in classic single split; do
  for w in 2 8; do
    PF_CG_VARIANT=$v timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/cg1_slab_${v}_$w.log 2>&1
    echo "$v world $w:"; tail -3 gpurun_out/cg1_slab_${v}_$w.log
  done
done
