#!/bin/bash
# compute-sanitizer over the device code paths with cross-CTA / cross-rank
# protocols: the fused Neumann-2 passes (two barriers per plane step,
# rotating shared-memory rings, last-CTA grid reductions) and a one-slab
# step (the slab plan's halo puts / flag waits and in-kernel allreduce
# talking to itself).  Several slabs sharing one device cannot run under
# the sanitizer: it serialises kernels, so ranks spinning on each other's
# flags time out (by design an error, not a hang).  Results -> gpurun_out/.
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
export CUDA_MODULE_LOADING=EAGER PF_NO_GRAPHS=1 PF_MAX_BATCH=4
SEL='tests/test_gpu_slab.py::test_slab_step_matches_single_domain[1] tests/test_gpu_neumann.py::test_neumann_matches_exact[shape0-True] tests/test_gpu_neumann.py::test_neumann_zero_and_converged_components'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest $SEL -m gpu -q -p no:cacheprovider --timeout 1400 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_$tool.log
  tail -n 4 gpurun_out/sanitize_$tool.log
done
