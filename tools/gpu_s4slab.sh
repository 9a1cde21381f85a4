#!/bin/bash
# slab decomposition cost with the Neumann-2 default + sanitizer over the staged multigrid cycle and the nm passes
mkdir -p gpurun_out/s4slab; cd $GRAFT_REPO_ROOT
for w in 1 2 8; do
  timeout 900 python tools/slab_overhead.py --world $w --steps 3 > gpurun_out/s4slab/slab_overhead_$w.log 2>&1
  echo "world $w exit $?"; tail -n 2 gpurun_out/s4slab/slab_overhead_$w.log
done
export CUDA_MODULE_LOADING=EAGER PF_NO_GRAPHS=1 PF_MAX_BATCH=4
SEL='tests/test_gpu_parity.py::test_multigrid_staged_coarse_cycle_matches_global tests/test_gpu_slab.py::test_slab_step_matches_single_domain[1] tests/test_gpu_neumann.py::test_neumann_matches_exact[shape0-True]'
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest $SEL -m gpu -q -p no:cacheprovider --timeout 1100 > gpurun_out/s4slab/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/s4slab/sanitize_$tool.log
  tail -n 3 gpurun_out/s4slab/sanitize_$tool.log
done
