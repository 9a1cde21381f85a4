#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
NM_ITERS=3 NM_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bi_nm --launch-skip 2 --launch-count 1 -o gpurun_out/nm_full3 -f python tools/dev/nm_profile.py 256,192,256 1 > gpurun_out/nm_ncu3.log 2>&1
tail -3 gpurun_out/nm_ncu3.log
