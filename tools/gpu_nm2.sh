#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/nm_profile.py > gpurun_out/nm_time2.log 2>&1
cat gpurun_out/nm_time2.log
timeout 900 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py -m gpu -q -s -x --timeout 300 > gpurun_out/nm2.log 2>&1
echo "nm exit $?" >> gpurun_out/nm2.log
tail -n 30 gpurun_out/nm2.log
NM_ITERS=3 NM_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bi_nm --launch-skip 2 --launch-count 2 -o gpurun_out/nm_full2 -f python tools/dev/nm_profile.py 256,192,256 1 > gpurun_out/nm_ncu2.log 2>&1
tail -3 gpurun_out/nm_ncu2.log
