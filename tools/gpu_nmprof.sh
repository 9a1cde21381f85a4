#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
python tools/dev/nm_profile.py > gpurun_out/nm_time.log 2>&1
PF_NO_NEUMANN=1 python tools/dev/nm_profile.py >> gpurun_out/nm_time.log 2>&1
cat gpurun_out/nm_time.log
NM_ITERS=3 NM_REPS=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_bi_nm --launch-skip 2 --launch-count 2 -o gpurun_out/nm_full -f python tools/dev/nm_profile.py 256,192,256 1 > gpurun_out/nm_ncu.log 2>&1
tail -5 gpurun_out/nm_ncu.log
