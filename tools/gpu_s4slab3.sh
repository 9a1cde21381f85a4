#!/bin/bash
mkdir -p gpurun_out/s4slab; cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_tiled.py tests/test_gpu_slab_ipc.py tests/test_gpu_graphs.py -m gpu -q --timeout 600 -x > gpurun_out/s4slab/test.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/s4slab/test.log
for w in 2 8; do
  timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/s4slab/slab_overhead_default_$w.log 2>&1
  echo "default world $w exit $?"; tail -n 2 gpurun_out/s4slab/slab_overhead_default_$w.log
done
