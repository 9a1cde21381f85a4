// cgstate.cuh -- device-resident Krylov state shared by the solver kernels
// and the multigrid kernels that fuse the CG z-sums into their last pass.
#pragma once

#include "common.cuh"

namespace pf {

struct CompState {
  double bnorm, tol_abs, res, rho, rho_new, alpha, omega, beta;
  // rho_next: r^.r of the next iteration, formed by the merged BiCGStab
  // passes from the st-pass sums (r^.s - omega r^.t) before r is
  double zbar, rz, xmean, true_res, bmean, rmean, tol, rho_next;
  int32_t iter, maxiter, done, converged, fail, zero_rhs, pending, active;
  // brk_next: rho_next or omega vanished -- a breakdown unless the update
  // that follows converges
  // xr_applied: the Neumann-2 light pass (k_nm_xr) already made the x/r
  // update the next merged pass would make
  int32_t project_x, brk_next, xr_applied, pad2[5];
};

struct SolverState {
  CompState c[3];
  int32_t all_done, ncomp, precond, zero_mean;
  int32_t pad[12];
};

static_assert(sizeof(SolverState) <= 8 * kWsSolver, "solver state too big");

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// z-bar, r.z and beta from the sums (sum z, sum r.z, sum r); `initial`
// seeds rz for the first direction (S/linalg.py:146-149 / 162-168)
__device__ __forceinline__ void cg_fin_z(SolverState *st, double sz,
                                         double srz, double sr, double n,
                                         bool initial) {
  CompState &c = st->c[0];
  c.zbar = st->zero_mean ? sz / n : 0.0;
  const double rz_new = srz - c.zbar * sr;
  if (initial) {
    c.rz = rz_new;
    return;
  }
  if (!finite(rz_new) || c.rz == 0.0) {
    c.fail = 1;
    c.done = 1;
    st->all_done = 1;
    return;
  }
  c.beta = rz_new / c.rz;
  c.rz = rz_new;
  if (c.iter >= c.maxiter) {
    c.done = 1;
    st->all_done = 1;
  }
}

// optional fusion of the CG z-sums into the multigrid's final pass
struct CgFuse {
  SolverState *st;  // null: no fusion
  double *partials;
  unsigned *counter;
  int initial;
  // st null: a reduction of the caller's follows the application on the
  // stream (k_cg1_spmv), which every rank reaches only after its inverse
  // transposes' peer loads -- the spectral closing barrier is implied
  int caller_closes = 0;
};

}  // namespace pf
