#!/bin/bash
# ncu --set full captures of the step's main kernels (one launch each, the
# details page exported to CSV; the reports themselves stay on the box) and
# the launch list of one C4 step with DRAM bytes
mkdir -p gpurun_out/ncu; cd $GRAFT_REPO_ROOT
i=0
for k in "k_bi_tiled<true, 0, 2, false>" "k_bi_tiled<true, 1, 2, false>" "k_bi_xr<false>" "k_cg_tiled<0>" "k_cg_update_pt" "k_spec_ysolve" "k_spec_inv_z16" "k_spec_fwd_z16" "k_spec_x16" "k_bwd_h_cell" "k_h_stage" "k_assemble_momentum"; do
  i=$((i+1))
  tag=$(printf "%02d_%s" $i "$(echo "$k" | tr -cd 'a-z0-9_')")
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:$k" --launch-count 1 -o /tmp/$tag -f python tools/dev/step_launches.py > /tmp/$tag.log 2>&1
  ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/ncu/$tag.csv 2>/dev/null
  echo "$tag $? $(grep -c '' gpurun_out/ncu/$tag.csv)"
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches_c4_final.csv python tools/dev/step_launches.py > gpurun_out/step_final.log 2>&1
tail -1 gpurun_out/step_final.log
du -sh gpurun_out
