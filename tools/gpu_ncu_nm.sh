#!/bin/bash
# ncu --set full of the Neumann-2 passes of one C4 step (details + source pages as CSV)
mkdir -p gpurun_out/ncu_nm; cd $GRAFT_REPO_ROOT
i=0
for k in "k_bi_nm<.bool.1, .int.3, .bool.0" "k_bi_nm<.bool.0, .int.3, .bool.0" "k_bi_nm<.bool.1, .int.1, .bool.0" "k_bi_nm<.bool.0, .int.1, .bool.0"; do
  i=$((i+1))
  tag=$(printf "%02d_%s" $i "$(echo "$k" | tr -cd 'a-z0-9_' | sed 's/bool//g; s/int//g')")
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:$k" --launch-count 1 -o /tmp/$tag -f python tools/dev/step_launches.py > gpurun_out/ncu_nm/$tag.log 2>&1
  echo "$tag ncu $?"
  ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/ncu_nm/$tag.csv 2>/dev/null
  ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_nm/${tag}_sass.csv 2>/dev/null
  ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/ncu_nm/${tag}_raw.csv 2>/dev/null
  echo "$tag $(grep -c '' gpurun_out/ncu_nm/$tag.csv) $(du -sh gpurun_out/ncu_nm/${tag}_sass.csv)"
done
du -sh gpurun_out
