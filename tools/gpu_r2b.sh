#!/bin/bash
# GPU-box: Neumann-2 BiCGStab tests, C4 bench with and without it, the
# 2D config bench lines, then the whole gpu tier
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_tiled.py -m gpu -q -s --timeout 300 > gpurun_out/nm.log 2>&1
echo "nm exit $?" >> gpurun_out/nm.log
tail -n 30 gpurun_out/nm.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_nm.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c4_nm.log
PF_NO_NEUMANN=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_jac.log 2>&1
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?" >> gpurun_out/bench_$c.log
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for f in bench_c4_nm bench_c4_jac bench_c1 bench_c2 bench_c3; do echo "== $f"; grep '^{' gpurun_out/$f.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{})
    print(d.get('value'), d.get('ms_per_step'), d.get('iterations_per_step'), r.get('kernel'), r.get('frac'), (d.get('e2e') or {}).get('value'))"; tail -n 3 gpurun_out/$f.log | cut -c1-300; done
tail -n 15 gpurun_out/pytest_gpu.log
