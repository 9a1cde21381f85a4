#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "multigrid or mg or cavity" > gpurun_out/mgst_test.log 2>&1
echo "pytest exit $?"; tail -n 3 gpurun_out/mgst_test.log
for st in 1 0 1 0; do
for c in c1 c2; do
if [ $st == 0 ]; then export PF_MG_NO_STAGE=1; else unset PF_MG_NO_STAGE; fi
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mgst_${c}_$st.log 2>&1
grep '^{' gpurun_out/mgst_${c}_$st.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c staged=$st', round(d['value'],3), round(d['ms_per_step'],2), d['iterations_per_step'])" || tail -3 gpurun_out/mgst_${c}_$st.log
done; done
unset PF_MG_NO_STAGE
bash tools/gpu_step_ncu.sh c1 s4st > /dev/null 2>&1; head -12 gpurun_out/launches_c1_s4st.md; tail -1 gpurun_out/launches_c1_s4st.md
