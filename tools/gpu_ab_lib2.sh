#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py tests/test_gpu_slab.py -m gpu -q --timeout 600 -x > gpurun_out/ab2_test.log 2>&1
echo "pytest exit $?"; tail -n 3 gpurun_out/ab2_test.log
bash tools/gpu_ab_lib.sh
