#!/bin/bash
mkdir -p gpurun_out/s4slab; cd $GRAFT_REPO_ROOT
for w in 1 2 8; do
  PF_MOMENTUM_PRECOND=jacobi timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/s4slab/slab_overhead_jacobi_$w.log 2>&1
  echo "jacobi world $w exit $?"; tail -n 2 gpurun_out/s4slab/slab_overhead_jacobi_$w.log
  timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/s4slab/slab_overhead_nm_$w.log 2>&1
  echo "nm world $w exit $?"; tail -n 2 gpurun_out/s4slab/slab_overhead_nm_$w.log
done
