#!/bin/bash
mkdir -p gpurun_out/ncu; cd $GRAFT_REPO_ROOT
i=0
for k in 'k_bi_tiled<\(bool\)1, \(int\)0, \(int\)2, \(bool\)0>' 'k_bi_tiled<\(bool\)1, \(int\)1, \(int\)2, \(bool\)0>' 'k_bi_tiled<\(bool\)0, \(int\)2, \(int\)2, \(bool\)0>' 'k_bi_tiled<\(bool\)1, \(int\)3, \(int\)2, \(bool\)0>' 'k_bi_xr<\(bool\)0>' 'k_cg_tiled<\(int\)0>' 'k_cg_tiled<\(int\)1>'; do
  i=$((i+1))
  tag=$(printf "%02d_%s" $i "$(echo "$k" | tr -cd 'a-z_0-9' )")
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:$k" --launch-count 1 -o /tmp/$tag -f python tools/dev/step_launches.py > /tmp/$tag.log 2>&1
  ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/ncu/$tag.csv 2>/dev/null
  echo "$tag $(grep -c '' gpurun_out/ncu/$tag.csv)"; tail -2 /tmp/$tag.log | head -1
done
