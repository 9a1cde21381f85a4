// spectral.cuh -- spectral preconditioner for the pressure operator of a
// box whose X and Z axes are periodic and uniformly spaced (the channel).
//
// On such a grid the pressure operator K (S/piso.py:395-412) has face
// weights that are functions of Y alone up to the A^-1 weighting, which
// varies across an XZ plane only through the advective part of the momentum
// diagonal (relative spread ~1e-4 in the channel).  The preconditioner is
// the exact inverse of the XZ-plane-averaged operator:
//
//   real FFT along Z  ->  complex FFT along X  ->  per wavenumber pair a
//   tridiagonal solve along Y  ->  inverse FFTs,
//
// with the singular (0, 0) mode pinned (the CG projects to zero mean).  It
// is a fixed SPD operator on the zero-mean subspace, so CG keeps its
// guarantees and converges to the same discrete solution as with the
// reference's ILU(0) (S/linalg.py:88-108) -- in 2-3 iterations instead of
// tens.
//
// Layout: the work array is (Y, kz, kx) complex, kx fastest, so the X
// transforms read contiguous lines and the Y solve is coalesced across
// wavenumbers (one thread per real / imaginary part of a column).
#pragma once

#include "cgstate.cuh"
#include "comm.h"
#include "common.cuh"

namespace pf {

// true when the canonical box admits the spectral solve: periodic Z (and X
// in 3D) of power-of-two length 4..1024, walled Y
bool spec_ok(int dim, int sx, int sy, int sz, int px, int pz);
// bytes of the spectral arrays (beyond level 0's face weights)
int64_t spec_bytes(const SpecPlan &sp);
void spec_plan(SpecPlan &sp, int sx, int sy, int sz);
// slab decomposition of the X axis over `world` ranks (see SpecPlan)
void spec_slab_plan(SpecPlan &sp, int nxl, int x0, int rank, int world);
// bytes of this rank's transposed spectrum (lives in the comm's symmetric
// buffer so peers can store / load it), and its binding after attach
int64_t spec_slab_bytes(const SpecPlan &sp);
void spec_slab_bind(SpecPlan &sp, const CommHost &c);
// carve the arrays from `base`; returns the first byte past them
char *spec_bind(SpecPlan &sp, char *base);
// plane means of the level-0 face weights, twiddles, eigenvalues
int spec_setup(const MgLevel &l0, const SpecPlan &sp, cudaStream_t s,
               const int *done, const Plan *pl);
// z = M^-1 r; `ev` (6 events) brackets the five passes; `fuse` folds the CG
// z-sums into the last pass
int spec_apply(const MgLevel &l0, const SpecPlan &sp, const double *r,
               double *z, cudaStream_t s, const int *done, cudaEvent_t *ev,
               const CgFuse *fuse, int red_blocks, const Plan *pl);

}  // namespace pf
