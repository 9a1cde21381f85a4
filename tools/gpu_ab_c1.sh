#!/bin/bash
# same-box A/B of two library builds on C1 / C2 (+ the gpu tier on build b)
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
L=paper_2505_16992_b200
cp $L/libpisob200_b.so $L/libpisob200.so
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/abc1_test.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/abc1_test.log
for v in a b a b; do
  cp $L/libpisob200_$v.so $L/libpisob200.so
  for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abc1_${c}_$v.log 2>&1
  grep '^{' gpurun_out/abc1_${c}_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c $v', round(d['value'],3), round(d['ms_per_step'],2), d['gpu_launches'], d['iterations_per_step'])"
  done
done
