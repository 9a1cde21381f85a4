#!/bin/bash
# ncu --set full captures of the step's main kernels (one launch each) and
# the launch list of one C4 step
mkdir -p gpurun_out/ncu; cd $GRAFT_REPO_ROOT
i=0
for k in "k_bi_tiled<true, 0, 2, false>" "k_bi_tiled<true, 1, 2, false>" "k_bi_xr<false>" "k_cg_spmv_pt" "k_cg_update_pt" "k_spec_ysolve" "k_spec_inv_z16" "k_spec_fwd_z16" "k_bwd_h_cell"; do
  i=$((i+1))
  tag=$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:$k" --launch-count 1 -o gpurun_out/ncu/$i_$tag -f python tools/dev/step_launches.py > gpurun_out/ncu/$tag.log 2>&1
  echo "$tag $?"
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches_c4_final.csv python tools/dev/step_launches.py > gpurun_out/step_final.log 2>&1
tail -2 gpurun_out/step_final.log
