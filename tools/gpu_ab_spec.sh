#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
L=paper_2505_16992_b200
cp $L/libpisob200_b.so $L/libpisob200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q --timeout 600 -x -k "spectral or channel or c4" > gpurun_out/abspec_test.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/abspec_test.log
bash tools/gpu_ab_lib.sh 2>&1 | grep -v "k_bi_nm\|k_cg_update"
