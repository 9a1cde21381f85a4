#!/bin/bash
# Neumann-2 light finishing pass: tests + same-box A/B bench
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py tests/test_gpu_graphs.py -q -x --timeout 600 > gpurun_out/nml_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/nml_tests.log
tail -3 gpurun_out/nml_tests.log
bash tools/gpu_nmab.sh
