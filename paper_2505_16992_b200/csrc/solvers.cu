// solvers.cu -- device-resident Krylov solvers with the reference semantics.
//
// CG with zero-mean projection (S/linalg.py:136-170) and BiCGStab
// (S/linalg.py:173-212) behind the verification/fallback wrapper
// (S/linalg.py:215-255).  The preconditioner is Jacobi (ILU(0), the
// reference's choice, is a sequential triangular solve with ~2(nx+ny+nz)
// dependent wavefronts and no place on a 148-SM GPU, SURVEY.md §7 hard part
// 1); results agree with the reference to solver tolerance, iteration counts
// differ and are reported.
//
// Every iteration is a short chain of fused streaming kernels; each fused
// reduction finishes in the last CTA to arrive, which also evaluates the
// recurrence scalars (alpha, beta, omega, convergence) into a device-side
// state block.  The host only polls that block every few iterations, so the
// GPU never waits on a host round trip per iteration.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>

#include "cgstate.cuh"
#include "common.cuh"
#include "mg.cuh"

namespace pf {

// ---------------------------------------------------------------------------
// stencil application  y_i = sum_j A_ij x_j  (transposed: A_ji)

template <class V, bool kTrans>
__device__ __forceinline__ double apply_row(const V &v, int32_t i,
                                            const Face (&fc)[2 * V::kDim],
                                            const double *__restrict__ a,
                                            const double *__restrict__ x) {
  constexpr int D = V::kDim;
  const int64_t n = v.n;
  double acc = a[i] * x[i];
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    if (fc[f].nb < 0) continue;
    const double coef =
        kTrans ? a[(int64_t)(1 + back_face(fc[f], f & 1)) * n + fc[f].nb]
               : a[(int64_t)(1 + f) * n + i];
    acc += coef * x[fc[f].nb];
  }
  return acc;
}

template <class V>
__device__ __forceinline__ void load_faces(const V &v, int32_t i,
                                           Face (&fc)[2 * V::kDim]) {
  const auto cell = v.topo.cell(i);
#pragma unroll
  for (int f = 0; f < 2 * V::kDim; ++f) fc[f] = v.topo.face(cell, f);
}

__device__ __forceinline__ double prec(int precond, const double *__restrict__ a,
                                       int32_t i, double r) {
  return precond ? r / a[i] : r;
}

#define GRID_LOOP(i, n)                                                  \
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (n);       \
       i += gridDim.x * blockDim.x)

// ===========================================================================
// CG

__global__ void k_cg_reset(SolverState *st, int maxiter, int precond,
                           int zero_mean, double tol, int fresh) {
  CompState &c = st->c[0];
  if (fresh) {
    c.bnorm = 0.0;
    c.bmean = 0.0;
    c.zero_rhs = 0;
  }
  c.tol = tol;
  c.iter = 0;
  c.maxiter = maxiter;
  c.done = c.zero_rhs;
  c.converged = c.zero_rhs;
  c.fail = 0;
  c.project_x = 0;
  c.res = 0.0;
  c.true_res = 0.0;
  c.active = 1;
  st->all_done = c.done;
  st->ncomp = 1;
  st->precond = precond;
  st->zero_mean = zero_mean;
}

__global__ void __launch_bounds__(kBlock)
    k_cg_bsum(const double *__restrict__ b, double bs, Rng rg,
              SolverState *st, double *partials, unsigned *counter) {
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) acc[0] += bs * b[i];
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot))
    st->c[0].bmean = st->zero_mean ? tot[0] / rg.ng : 0.0;
}

__global__ void __launch_bounds__(kBlock)
    k_cg_bproj(const double *__restrict__ b, double bs,
               double *__restrict__ bp, Rng rg, SolverState *st,
               double *partials, unsigned *counter) {
  const double mean = st->c[0].bmean;
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) {
    const double x = bs * b[i] - mean;
    bp[i] = x;
    acc[0] += x * x;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.bnorm = sqrt(tot[0]);
    c.tol_abs = c.tol * c.bnorm;
    if (c.bnorm == 0.0) {
      c.zero_rhs = 1;
      c.done = 1;
      c.converged = 1;
      st->all_done = 1;
    }
  }
}

// r = bp - A x, accumulate sum r
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_cg_resid(V v, const double *__restrict__ a, const double *__restrict__ bp,
               const double *__restrict__ x, double *__restrict__ r,
               SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  double acc[1] = {0.0};
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    const double ri = bp[i] - apply_row<V, false>(v, i, fc, a, x);
    r[i] = ri;
    acc[0] += ri;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot))
    st->c[0].rmean = st->zero_mean ? tot[0] / v.ng : 0.0;
}

// z value of cell i: the multigrid output vector, or M r pointwise
__device__ __forceinline__ double zval(int pc, const double *__restrict__ a,
                                       const double *__restrict__ z,
                                       int32_t i, double ri) {
  return pc == 2 ? z[i] : prec(pc, a, i, ri);
}

// r -= mean(r); |r|; (pointwise preconditioners) z sums
__global__ void __launch_bounds__(kBlock)
    k_cg_rproj(const double *__restrict__ a, double *__restrict__ r, Rng rg,
               SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  const double rmean = st->c[0].rmean;
  const int pc = st->precond;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
    const double ri = r[i] - rmean;
    r[i] = ri;
    acc[0] += ri * ri;
    if (pc != 2) {
      const double zi = prec(pc, a, i, ri);
      acc[1] += zi;
      acc[2] += ri * zi;
      acc[3] += ri;
    }
  }
  double tot[4];
  if (grid_reduce<4>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.res = sqrt(tot[0]);
    if (c.res <= c.tol_abs) {
      c.converged = 1;
      c.done = 1;
      st->all_done = 1;
      return;
    }
    if (pc != 2) cg_fin_z(st, tot[1], tot[2], tot[3], rg.ng, true);
  }
}

// z sums for a stored z (multigrid), then beta
__global__ void __launch_bounds__(kBlock)
    k_cg_zsum(const double *__restrict__ r, const double *__restrict__ z,
              Rng rg, int initial, SolverState *st, double *partials,
              unsigned *counter) {
  if (st->all_done) return;
  double acc[3] = {0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
    const double ri = r[i], zi = z[i];
    acc[0] += zi;
    acc[1] += ri * zi;
    acc[2] += ri;
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot))
    cg_fin_z(st, tot[0], tot[1], tot[2], rg.ng, initial != 0);
}

__global__ void __launch_bounds__(kBlock)
    k_cg_pinit(const double *__restrict__ a, const double *__restrict__ r,
               const double *__restrict__ z, double *__restrict__ p,
               Rng rg, const SolverState *st) {
  if (st->all_done) return;
  const double zbar = st->c[0].zbar;
  const int pc = st->precond;
  RANGE_LOOP(i, rg) p[i] = zval(pc, a, z, i, r[i]) - zbar;
}

// q = A p; p.q -> alpha
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_cg_spmv(V v, const double *__restrict__ a, const double *__restrict__ p,
              double *__restrict__ q, SolverState *st, double *partials,
              unsigned *counter) {
  if (st->all_done) return;
  double acc[1] = {0.0};
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    const double qi = apply_row<V, false>(v, i, fc, a, p);
    q[i] = qi;
    acc[0] += p[i] * qi;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.iter += 1;
    const double pap = tot[0];
    if (!finite(pap) || fabs(pap) < DBL_MIN) {
      c.fail = 1;
      c.done = 1;
      st->all_done = 1;
      return;
    }
    c.alpha = c.rz / pap;
  }
}

// q = K p on the multigrid level-0 face form (d face weights per cell, the
// diagonal as their sum): 40 B/cell in 3D instead of the 72 B/cell of the
// (2d+1)-row stencil
__global__ void __launch_bounds__(kBlock)
    k_cg_spmv_faces(MgLevel L, Rng rg, const double *__restrict__ p,
                    double *__restrict__ q, SolverState *st, double *partials,
                    unsigned *counter) {
  if (st->all_done) return;
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) {
    const Cell3 c = decode(L, i);
    const Nbhd b = nbhd(L, c);
    const double qi = kx(b, i, p);
    q[i] = qi;
    acc[0] += p[i] * qi;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.iter += 1;
    const double pap = tot[0];
    if (!finite(pap) || fabs(pap) < DBL_MIN) {
      c.fail = 1;
      c.done = 1;
      st->all_done = 1;
      return;
    }
    c.alpha = c.rz / pap;
  }
}

// x += alpha p; r -= alpha q; convergence; (pointwise M) z sums and beta
__global__ void __launch_bounds__(kBlock)
    k_cg_update(const double *__restrict__ a, const double *__restrict__ p,
                const double *__restrict__ q, double *__restrict__ x,
                double *__restrict__ r, Rng rg, SolverState *st,
                double *partials, unsigned *counter) {
  if (st->all_done) return;
  const double alpha = st->c[0].alpha;
  const int pc = st->precond;
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
    const double xi = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    x[i] = xi;
    r[i] = ri;
    acc[0] += ri * ri;
    acc[4] += xi;
    if (pc != 2) {
      const double zi = prec(pc, a, i, ri);
      acc[1] += zi;
      acc[2] += ri * zi;
      acc[3] += ri;
    }
  }
  double tot[5];
  if (grid_reduce<5>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.res = sqrt(tot[0]);
    if (c.res <= c.tol_abs) {
      c.converged = 1;
      c.done = 1;
      c.project_x = st->zero_mean;
      c.xmean = st->zero_mean ? tot[4] / rg.ng : 0.0;
      st->all_done = 1;
      return;
    }
    if (pc != 2) cg_fin_z(st, tot[1], tot[2], tot[3], rg.ng, false);
  }
}

// k_cg_update for the fused direction update (cg_tiled.cuh): p is the
// direction the last k_cg_spmv_pt wrote, P[(c.iter - 1) & 1]
__global__ void __launch_bounds__(kBlock)
    k_cg_update_pt(const double *__restrict__ p0, const double *__restrict__ p1,
                   const double *__restrict__ q, double *__restrict__ x,
                   double *__restrict__ r, Rng rg, SolverState *st,
                   double *partials, unsigned *counter) {
  if (st->all_done) return;
  const double *__restrict__ p = ((st->c[0].iter - 1) & 1) ? p1 : p0;
  const double alpha = st->c[0].alpha;
  double acc[2] = {0.0, 0.0};
  RANGE_LOOP(i, rg) {
    const double xi = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    x[i] = xi;
    r[i] = ri;
    acc[0] += ri * ri;
    acc[1] += xi;
  }
  double tot[2];
  if (grid_reduce<2>(acc, partials, counter, tot)) {
    CompState &c = st->c[0];
    c.res = sqrt(tot[0]);
    if (c.res <= c.tol_abs) {
      c.converged = 1;
      c.done = 1;
      c.project_x = st->zero_mean;
      c.xmean = st->zero_mean ? tot[1] / rg.ng : 0.0;
      st->all_done = 1;
    }
  }
}

__global__ void __launch_bounds__(kBlock)
    k_cg_pupdate(const double *__restrict__ a, const double *__restrict__ r,
                 const double *__restrict__ z, double *__restrict__ p,
                 Rng rg, const SolverState *st) {
  if (st->all_done) return;
  const double beta = st->c[0].beta, zbar = st->c[0].zbar;
  const int pc = st->precond;
  RANGE_LOOP(i, rg) p[i] = beta * p[i] + (zval(pc, a, z, i, r[i]) - zbar);
}

__global__ void __launch_bounds__(kBlock)
    k_cg_finish(double *__restrict__ x, Rng rg, const SolverState *st) {
  const CompState &c = st->c[0];
  if (c.zero_rhs) {
    RANGE_LOOP(i, rg) x[i] = 0.0;
  } else if (c.project_x) {
    const double m = c.xmean;
    RANGE_LOOP(i, rg) x[i] -= m;
  }
}

// |bp - A x|
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_true_res(V v, const double *__restrict__ a, int trans, int ncomp,
               const double *__restrict__ b, const double *__restrict__ x,
               SolverState *st, double *partials, unsigned *counter) {
  double acc[3] = {0.0, 0.0, 0.0};
  const int64_t n = v.n;
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    for (int q = 0; q < ncomp; ++q) {
      const double ax = trans ? apply_row<V, true>(v, i, fc, a, x + q * n)
                              : apply_row<V, false>(v, i, fc, a, x + q * n);
      const double d = b[q * n + i] - ax;
      acc[q] += d * d;
    }
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot)) {
    for (int q = 0; q < ncomp; ++q) st->c[q].true_res = sqrt(tot[q]);
  }
}

// ===========================================================================
// BiCGStab on ncomp right-hand sides sharing one matrix
//
// Three fused passes per iteration (S/linalg.py:183-211 restated):
//   pv: p = r + beta (p - omega v) and v = A M^-1 p in one sweep -- the
//       stencil gathers the neighbours' r, p, v and forms their p on the fly,
//       so neither p nor phat makes a separate trip through HBM; r^.v -> alpha
//   st: s = r - alpha v (on the fly again) and t = A M^-1 s;
//       |s|, t.t, t.s -> early exit / omega
//   xr: x += M^-1 (alpha p + omega s); r = s - omega t; |r|, r^.r -> beta
// p and v are ping-ponged by iteration parity (the stencil of cell i reads
// its neighbours' old p while i writes its new one).  M is Jacobi: M^-1 y is
// y_j / A_jj, evaluated where the value is gathered.

struct BiVecs {
  double *r, *rhat, *t;   // each (ncomp, n)
  double *p[2], *v[2];    // ping-pong by iteration parity
  double *dinv;           // (n) Jacobi: 1 / A_ii (ones when unpreconditioned)
  double *rb[2] = {nullptr, nullptr};  // merged Neumann-2 passes: r by
                                       // parity (rb[0] = r)
  double *z = nullptr;    // Neumann-2: the preconditioned iterate
};

__global__ void k_bi_reset(SolverState *st, int ncomp, int maxiter,
                           int precond, double tol, int fresh,
                           unsigned active_mask) {
  st->ncomp = ncomp;
  st->precond = precond;
  st->zero_mean = 0;
  int all = 1;
  for (int q = 0; q < 3; ++q) {
    CompState &c = st->c[q];
    if (fresh) {
      c.bnorm = 0.0;
      c.zero_rhs = 0;
    }
    c.active = (q < ncomp) && ((active_mask >> q) & 1u);
    c.tol = tol;
    c.iter = 0;
    c.maxiter = maxiter;
    c.done = !c.active || c.zero_rhs;
    c.converged = c.active && c.zero_rhs;
    c.fail = 0;
    c.pending = 0;
    c.xr_applied = 0;
    c.res = 0.0;
    c.true_res = 0.0;
    if (!c.done) all = 0;
  }
  st->all_done = all;
}

__global__ void __launch_bounds__(kBlock)
    k_bi_bnorm(const double *__restrict__ b, int32_t n, Rng rg, SolverState *st,
               double *partials, unsigned *counter) {
  const int nc = st->ncomp;
  double acc[3] = {0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
    for (int q = 0; q < nc; ++q) {
      const double x = b[(int64_t)q * n + i];
      acc[q] += x * x;
    }
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot)) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      c.bnorm = sqrt(tot[q]);
      c.tol_abs = c.tol * c.bnorm;
      if (c.bnorm == 0.0 && c.active) {
        c.zero_rhs = 1;
        c.done = 1;
        c.converged = 1;
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  }
}

// r = b - A x; rhat = r; p = v = 0 (parity-0 buffers)
template <class V, bool kTrans>
__global__ void __launch_bounds__(kBlock)
    k_bi_init(V v, const double *__restrict__ a, const double *__restrict__ b,
              const double *__restrict__ x, BiVecs w, SolverState *st,
              double *partials, unsigned *counter) {
  if (st->all_done) return;
  const int nc = st->ncomp;
  const int64_t n = v.n;
  int act[3];
  for (int q = 0; q < 3; ++q) act[q] = q < nc && !st->c[q].done;
  double acc[3] = {0.0, 0.0, 0.0};
  const int pc = st->precond;
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    w.dinv[i] = pc ? 1.0 / a[i] : 1.0;
    for (int q = 0; q < nc; ++q) {
      if (!act[q]) continue;
      const int64_t o = q * n;
      const double ri = b[o + i] - apply_row<V, kTrans>(v, i, fc, a, x + o);
      w.r[o + i] = ri;
      w.rhat[o + i] = ri;
      w.p[0][o + i] = 0.0;
      w.v[0][o + i] = 0.0;
      acc[q] += ri * ri;
    }
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot)) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (act[q]) {
        c.res = sqrt(tot[q]);
        if (c.res <= c.tol_abs) {
          c.converged = 1;
          c.done = 1;
        } else {
          c.rho = c.alpha = c.omega = 1.0;
          c.iter = 1;
          c.rho_new = tot[q];
          if (fabs(c.rho_new) < DBL_MIN || fabs(c.omega) < DBL_MIN) {
            c.fail = 1;
            c.done = 1;
          } else {
            c.beta = (c.rho_new / c.rho) * (c.alpha / c.omega);
          }
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  }
}

// y_i = sum_j A_ij g(j) (transposed: A_ji) for NC right-hand sides at once;
// g(q, j) is the preconditioned input value of component q at cell j.
template <class V, bool kTrans, class G>
__device__ __forceinline__ void apply_rows(const V &v, int32_t i,
                                           const Face (&fc)[2 * V::kDim],
                                           const double *__restrict__ a,
                                           const int (&act)[3], int nc,
                                           G &&g, double (&y)[3]) {
  constexpr int D = V::kDim;
  const int64_t n = v.n;
  const double aii = a[i];
#pragma unroll
  for (int q = 0; q < 3; ++q)
    y[q] = (q < nc && act[q]) ? aii * g(q, i) : 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int32_t j = fc[f].nb;
    if (j < 0) continue;
    const double coef =
        kTrans ? a[(int64_t)(1 + back_face(fc[f], f & 1)) * n + j]
               : a[(int64_t)(1 + f) * n + i];
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (q < nc && act[q]) y[q] += coef * g(q, j);
  }
}

// pass pv: p' = r + beta (p - omega v); v' = A M^-1 p'; r^.v' -> alpha
template <class V, bool kTrans>
__global__ void __launch_bounds__(kBlock)
    k_bi_pv(V v, const double *__restrict__ a, BiVecs w, int par,
            SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  const int nc = st->ncomp, pc = st->precond;
  const int64_t n = v.n;
  int act[3];
  double beta[3], omega[3];
  _Pragma("unroll") for (int q = 0; q < 3; ++q) {
    act[q] = q < nc && !st->c[q].done;
    beta[q] = q < nc ? st->c[q].beta : 0.0;
    omega[q] = q < nc ? st->c[q].omega : 0.0;
  }
  const double *__restrict__ r = w.r;
  const double *__restrict__ dinv = w.dinv;
  const double *__restrict__ p0 = w.p[par];
  const double *__restrict__ v0 = w.v[par];
  double *__restrict__ p1 = w.p[par ^ 1];
  double *__restrict__ v1 = w.v[par ^ 1];
  double acc[3] = {0.0, 0.0, 0.0};
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    auto pnew = [&](int q, int32_t j) {
      const int64_t o = q * n + j;
      return r[o] + beta[q] * (p0[o] - omega[q] * v0[o]);
    };
    auto g = [&](int q, int32_t j) { return pnew(q, j) * dinv[j]; };
    double y[3];
    apply_rows<V, kTrans>(v, i, fc, a, act, nc, g, y);
    _Pragma("unroll") for (int q = 0; q < 3; ++q) {
      if (q >= nc) break;
      if (!act[q]) continue;
      const int64_t o = q * n + i;
      p1[o] = pnew(q, i);
      v1[o] = y[q];
      acc[q] += w.rhat[o] * y[q];
    }
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot)) {
    int all = 1;
    _Pragma("unroll") for (int q = 0; q < 3; ++q) {
      if (q >= nc) break;
      CompState &c = st->c[q];
      if (act[q]) {
        if (fabs(tot[q]) < DBL_MIN) {
          c.fail = 1;
          c.done = 1;
        } else {
          c.alpha = c.rho_new / tot[q];
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  }
}

// pass st: s = r - alpha v'; t = A M^-1 s; |s| (early exit), t.t, t.s
template <class V, bool kTrans>
__global__ void __launch_bounds__(kBlock)
    k_bi_st(V v, const double *__restrict__ a, BiVecs w, int par,
            SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  const int nc = st->ncomp, pc = st->precond;
  const int64_t n = v.n;
  int act[3];
  double alpha[3];
  _Pragma("unroll") for (int q = 0; q < 3; ++q) {
    act[q] = q < nc && !st->c[q].done;
    alpha[q] = q < nc ? st->c[q].alpha : 0.0;
  }
  const double *__restrict__ r = w.r;
  const double *__restrict__ dinv = w.dinv;
  const double *__restrict__ v1 = w.v[par ^ 1];
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  RANGE_LOOP(i, v.rng()) {
    Face fc[2 * V::kDim];
    load_faces(v, i, fc);
    auto sval = [&](int q, int32_t j) {
      const int64_t o = q * n + j;
      return r[o] - alpha[q] * v1[o];
    };
    auto g = [&](int q, int32_t j) { return sval(q, j) * dinv[j]; };
    double y[3];
    apply_rows<V, kTrans>(v, i, fc, a, act, nc, g, y);
    _Pragma("unroll") for (int q = 0; q < 3; ++q) {
      if (q >= nc) break;
      if (!act[q]) continue;
      const double si = sval(q, i);
      w.t[q * n + i] = y[q];
      acc[3 * q] += si * si;
      acc[3 * q + 1] += y[q] * y[q];
      acc[3 * q + 2] += y[q] * si;
    }
  }
  double tot[9];
  if (grid_reduce<9>(acc, partials, counter, tot)) {
    // all_done is deliberately left alone: k_bi_xr must still run to apply
    // the early-exit update x += alpha phat
    _Pragma("unroll") for (int q = 0; q < 3; ++q) {
      if (q >= nc) break;
      CompState &c = st->c[q];
      if (!act[q]) continue;
      c.res = sqrt(tot[3 * q]);
      if (c.res <= c.tol_abs) {
        c.converged = 1;
        c.done = 1;
        c.pending = 1;
      } else if (tot[3 * q + 1] < DBL_MIN) {
        c.fail = 1;
        c.done = 1;
      } else {
        c.omega = tot[3 * q + 2] / tot[3 * q + 1];
      }
    }
  }
}

// pass xr: pending comps: x += alpha phat.  active comps:
// x += alpha phat + omega shat; r = s - omega t; |r|, r^.r -> next beta.
// Two cells per thread with 128-bit loads and stores (the owned range is
// split into an even-aligned vector part and scalar edges).
//
// kZ (Neumann-2 passes): x is the preconditioned iterate z (x = x0 + M^-1 z
// is formed once at the end), so z += alpha p' + omega s with no division;
// zfirst: the first iteration's z starts from 0 (it is neither read nor
// memset).
template <bool kZ = false>
__global__ void __launch_bounds__(kBlock)
    k_bi_xr(const double *__restrict__ a, BiVecs w, int par,
            double *__restrict__ x, int32_t n, Rng rg, SolverState *st,
            double *partials, unsigned *counter, int zfirst = 0) {
  if (st->all_done) return;
  const int nc = st->ncomp;
  int act[3], pend[3];
  double alpha[3], omega[3];
  _Pragma("unroll") for (int q = 0; q < 3; ++q) {
    act[q] = q < nc && !st->c[q].done;
    pend[q] = q < nc && st->c[q].pending;
    alpha[q] = q < nc ? st->c[q].alpha : 0.0;
    omega[q] = q < nc ? st->c[q].omega : 0.0;
  }
  const double *__restrict__ p1 = w.p[par ^ 1];
  const double *__restrict__ v1 = w.v[par ^ 1];
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const bool z0 = kZ && zfirst;
  auto cell = [&](int32_t i) {
    const double di = kZ ? 1.0 : w.dinv[i];
    _Pragma("unroll") for (int q = 0; q < 3; ++q) {
      if (q >= nc) break;
      const int64_t o = (int64_t)q * n + i;
      if (z0 && (act[q] || pend[q])) x[o] = 0.0;
      if (pend[q]) x[o] += alpha[q] * (p1[o] * di);
      if (!act[q]) continue;
      const double phat = p1[o] * di;
      const double si = w.r[o] - alpha[q] * v1[o];
      const double shat = si * di;
      x[o] = x[o] + alpha[q] * phat + omega[q] * shat;
      const double ri = si - omega[q] * w.t[o];
      w.r[o] = ri;
      acc[2 * q] += ri * ri;
      acc[2 * q + 1] += w.rhat[o] * ri;
    }
  };
  // n even: component bases stay 16-byte aligned
  const int32_t v0 = (n & 1) ? rg.i1 : ((rg.i0 + 1) & ~1);
  const int32_t v1e = (n & 1) ? rg.i1 : (rg.i1 & ~1);
  const int32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t nth = gridDim.x * blockDim.x;
  const double *__restrict__ rr_ = w.r;
  const double *__restrict__ tt_ = w.t;
  const double *__restrict__ rh_ = w.rhat;
  const double *__restrict__ di_ = w.dinv;
  double *__restrict__ rw_ = w.r;
  for (int32_t k = v0 + 2 * tid; k + 1 < v1e; k += 2 * nth) {
    // every load of the three components first (the stores below cannot
    // then serialise them), then the updates
    const double2 di = kZ ? make_double2(1.0, 1.0)
                          : *reinterpret_cast<const double2 *>(di_ + k);
    double2 pp[3], xx[3], rr[3], vv[3], tt[3], rh[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q >= nc || !(act[q] || pend[q])) continue;
      const int64_t o = (int64_t)q * n + k;
      pp[q] = *reinterpret_cast<const double2 *>(p1 + o);
      xx[q] = z0 ? make_double2(0.0, 0.0)
                 : *reinterpret_cast<const double2 *>(x + o);
      if (!act[q]) continue;
      rr[q] = *reinterpret_cast<const double2 *>(rr_ + o);
      vv[q] = *reinterpret_cast<const double2 *>(v1 + o);
      tt[q] = *reinterpret_cast<const double2 *>(tt_ + o);
      rh[q] = *reinterpret_cast<const double2 *>(rh_ + o);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q >= nc || !(act[q] || pend[q])) continue;
      const int64_t o = (int64_t)q * n + k;
      double2 xn = xx[q];
      if (pend[q]) {
        xn.x += alpha[q] * (pp[q].x * di.x);
        xn.y += alpha[q] * (pp[q].y * di.y);
      }
      if (act[q]) {
        const double s0 = rr[q].x - alpha[q] * vv[q].x;
        const double s1 = rr[q].y - alpha[q] * vv[q].y;
        xn.x = xn.x + alpha[q] * (pp[q].x * di.x) + omega[q] * (s0 * di.x);
        xn.y = xn.y + alpha[q] * (pp[q].y * di.y) + omega[q] * (s1 * di.y);
        const double r0 = s0 - omega[q] * tt[q].x;
        const double r1 = s1 - omega[q] * tt[q].y;
        *reinterpret_cast<double2 *>(rw_ + o) = make_double2(r0, r1);
        acc[2 * q] += r0 * r0;
        acc[2 * q] += r1 * r1;
        acc[2 * q + 1] += rh[q].x * r0;
        acc[2 * q + 1] += rh[q].y * r1;
      }
      *reinterpret_cast<double2 *>(x + o) = xn;
    }
  }
  // scalar edges of the owned range
  if (tid == 0) {
    for (int32_t i = rg.i0; i < v0; ++i) cell(i);
    for (int32_t i = v1e; i < rg.i1; ++i) cell(i);
  }
  double tot[6];
  if (grid_reduce<6>(acc, partials, counter, tot)) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      c.pending = 0;
      if (act[q]) {
        c.res = sqrt(tot[2 * q]);
        if (c.res <= c.tol_abs) {
          c.converged = 1;
          c.done = 1;
        } else if (c.iter >= c.maxiter) {
          c.done = 1;
        } else {
          c.rho = c.rho_new;
          c.iter += 1;
          c.rho_new = tot[2 * q + 1];
          if (fabs(c.rho_new) < DBL_MIN || fabs(c.omega) < DBL_MIN) {
            c.fail = 1;
            c.done = 1;
          } else {
            c.beta = (c.rho_new / c.rho) * (c.alpha / c.omega);
          }
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  }
}

// ---------------------------------------------------------------------------
// Tiled stencil passes for 3D boxes (2.5D blocking).
//
// A CTA owns a TY x TZ column tile of the (Y, Z) plane and marches along X
// through a chunk of planes.  The preconditioned input g = M^-1 (r + beta
// (p - omega v)) (pass pv) or M^-1 (r - alpha v') (pass st) of every cell is
// formed ONCE: the centre column in registers for planes x-1, x, x+1, the
// current plane with its one-cell Y / Z halo in shared memory.  Every input
// array is then read from HBM once per cell (plus the thin halo and the two
// prologue planes of a chunk, from L2), instead of once per stencil point.

constexpr int kTZ = 32, kTY = 8, kTileThreads = kTZ * kTY;
constexpr int kXChunk = 64;  // X planes per tile (fewer on small boxes)

struct TileGeo {
  int32_t X, Y, Z;          // local box
  int32_t px, py, pz;       // periodic flags
  int32_t x0, x1;           // owned planes [x0, x1)
  int32_t ty_tiles, tz_tiles, chunks, ntiles;
  int32_t xc;               // X planes per chunk
};

__device__ __forceinline__ int32_t wrap(int32_t c, int32_t L, int32_t per,
                                        bool &ok) {
  if (c >= 0 && c < L) {
    ok = true;
    return c;
  }
  ok = per != 0;
  return c < 0 ? c + L : c - L;
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// all but the N most recent committed groups have landed
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Shared memory of the tiled passes: the raw inputs of two planes (tile +
// halo, filled by cp.async one plane ahead) and the preconditioned values
// g of two planes (double buffered, so a plane step needs one barrier).
constexpr int kRawArrays = 10;  // r x3, p x3, v x3, 1/A (pass st: r, v, 1/A)
constexpr int kTP = (kTY + 2) * (kTZ + 2);
struct TileSmem {
  double raw[2][kRawArrays][kTY + 2][kTZ + 2];
  double g[2][3][kTY + 2][kTZ + 2];
};
constexpr size_t kTileSmem = sizeof(TileSmem);

// Per-pass layout of the raw buffers: the pv pass stages 10 arrays two
// planes deep (71 KB, two CTAs per SM: a larger buffer shrinks the L1 the
// transposed neighbour gathers use and was measured slower); the lighter
// passes stage fewer arrays three planes deep, so a plane's loads have two
// plane steps to land
template <int MODE>
struct TileLayout {
  static constexpr int kStages = MODE == 0 ? 2 : 3;
  static constexpr int kArr = MODE == 0 ? 10 : MODE == 1 ? 7 : MODE == 4 ? 4 : 3;
  static constexpr int kDinv = MODE == 0 ? 9 : MODE == 1 ? 6 : 3;  // 1/A slot
  static constexpr size_t kBytes =
      sizeof(double) * (size_t)(kStages * kArr + 6) * kTP;
};

// MODE 0 (pass pv): g = (r + beta (p0 - omega v0)) / A, outputs p' (the
//                   undivided value), v' = A g, sums r^.v'.  `first` (the
//                   first iteration, p0 = v0 = 0): g = r / A, p0 and v0 are
//                   neither read nor (by MODE 2) written
// MODE 2 (init):    g = x, outputs r = r^ = b - A x, 1 / A; |r|, and |b|
//                   when the state has no |b| yet (a fresh solve: the
//                   separate k_bi_bnorm pass is folded in here)
// MODE 1 (pass st): g = (r - alpha v') / A, outputs t = A g, sums s.s, t.t,
//                   t.s
// MODE 3 (verify):  g = x, sums |b - A x|^2 of every component (runs after
//                   convergence too)
// MODE 4 (close):  g = z / A, x += g - A^-1 N g = x0 + M^-1 z (the
//                   Neumann-2 preconditioned iterate, bicg_nm.cuh); a
//                   one-stage stencil, so the efficient single-halo pass
//                   forms it (no reduction)
template <bool kTrans, int MODE, int kMinB = 1, bool kFirst = false>
__global__ void __launch_bounds__(kTileThreads, kMinB)
    k_bi_tiled(TileGeo tg, const double *__restrict__ a, BiVecs w, int par,
               int64_t n, SolverState *st, double *partials,
               unsigned *counter, const double *__restrict__ xin = nullptr,
               const double *__restrict__ bin = nullptr, int nverify = 0,
               double *__restrict__ xout = nullptr) {
  if (MODE != 3 && MODE != 4 && st->all_done) return;
  // the speculative close (nverify = 1) runs only once the solve ended
  if (MODE == 4 && nverify && !st->all_done) return;
  // compile-time: a runtime branch here slows the transposed pass ~15 %
  constexpr bool fresh = MODE == 0 && kFirst;
  constexpr int K = MODE == 1 ? 9 : MODE == 2 ? 6 : 3;
  constexpr bool kX = MODE >= 2;  // the input is the iterate x (or z) itself
  constexpr bool kZ = MODE == 4;  // ... divided by A (the close pass)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using TL = TileLayout<MODE>;
  constexpr int kStages = TL::kStages, kDs = TL::kDinv;
  using RawPlane = double[TL::kArr][kTY + 2][kTZ + 2];
  using GPlane = double[3][kTY + 2][kTZ + 2];
  RawPlane *raw = reinterpret_cast<RawPlane *>(smem_raw);
  GPlane *gbuf = reinterpret_cast<GPlane *>(
      smem_raw + sizeof(double) * (size_t)kStages * TL::kArr * kTP);
  // raw slot of plane x (x >= -1)
  auto slot = [](int32_t x) { return (x + kStages) % kStages; };
  const int nc = MODE == 3 ? nverify : st->ncomp;
  const int pc_on = st->precond;
  int act[3];
  double c0[3], c1[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    act[q] = q < nc && (MODE == 3 || !st->c[q].done);
    if (MODE == 4)  // the components that iterated and did not break down
      act[q] = q < nc && st->c[q].active && !st->c[q].zero_rhs &&
               st->c[q].iter > 0 && !st->c[q].fail;
    if (MODE == 0) {
      c0[q] = q < nc ? st->c[q].beta : 0.0;
      c1[q] = q < nc ? st->c[q].omega : 0.0;
    } else {
      c0[q] = q < nc ? st->c[q].alpha : 0.0;
      c1[q] = 0.0;
    }
  }
  const double *__restrict__ r = w.r;
  const double *__restrict__ dinv = w.dinv;
  const double *__restrict__ pin = MODE == 0 ? w.p[par] : nullptr;
  const double *__restrict__ vin = MODE == 0 ? w.v[par] : w.v[par ^ 1];
  double *__restrict__ pout = w.p[par ^ 1];
  double *__restrict__ vout = MODE == 0 ? w.v[par ^ 1] : w.t;
  const int64_t sX = (int64_t)tg.Y * tg.Z, sY = tg.Z;
  const int tz = threadIdx.x % kTZ, ty = threadIdx.x / kTZ;

  // async copy of the raw inputs of cell (x, y, z) into slot (sy, sz) of
  // raw buffer b; zeros outside a walled box
  auto issue = [&](int b, int32_t x, int32_t y, int32_t z, int sy, int sz) {
    bool okx, oky, okz;
    x = wrap(x, tg.X, tg.px, okx);
    y = wrap(y, tg.Y, tg.py, oky);
    z = wrap(z, tg.Z, tg.pz, okz);
    const bool ok = okx && oky && okz;
    const int64_t j = (int64_t)x * sX + (int64_t)y * sY + z;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q >= nc || !act[q]) continue;
      const int64_t o = q * n + j;
      if (kX) {
        if (ok)
          cp_async8(&raw[b][q][sy][sz], xin + o);
        else
          raw[b][q][sy][sz] = 0.0;
        continue;
      }
      if (ok) {
        cp_async8(&raw[b][q][sy][sz], r + o);
        if (!fresh) {
          cp_async8(&raw[b][3 + q][sy][sz], vin + o);
          if (MODE == 0) cp_async8(&raw[b][6 + q][sy][sz], pin + o);
        }
      } else {
        raw[b][q][sy][sz] = 0.0;
        raw[b][3 + q][sy][sz] = 0.0;
        if (MODE == 0) raw[b][6 + q][sy][sz] = 0.0;
      }
    }
    if (kX && !kZ) return;
    if (ok)
      cp_async8(&raw[b][kDs][sy][sz], dinv + j);
    else
      raw[b][kDs][sy][sz] = 0.0;
  };
  // g (and the undivided value) of slot (sy, sz) of raw buffer b
  auto G = [&](int b, int sy, int sz, double (&g)[3], double (&pv)[3]) {
    if (kZ) {
      const double dj = raw[b][kDs][sy][sz];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        pv[q] = (q < nc && act[q]) ? raw[b][q][sy][sz] : 0.0;
        g[q] = pv[q] * dj;
      }
      return;
    }
    if (kX) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        g[q] = pv[q] = (q < nc && act[q]) ? raw[b][q][sy][sz] : 0.0;
      }
      return;
    }
    const double dj = raw[b][kDs][sy][sz];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      g[q] = pv[q] = 0.0;
      if (q >= nc || !act[q]) continue;
      const double rr = raw[b][q][sy][sz];
      double val;
      if (fresh) {
        val = rr;  // r + beta (0 - omega 0)
      } else {
        const double vv = raw[b][3 + q][sy][sz];
        val = MODE == 0
                  ? rr + c0[q] * (raw[b][6 + q][sy][sz] - c1[q] * vv)
                  : rr - c0[q] * vv;
      }
      pv[q] = val;
      g[q] = val * dj;
    }
  };

  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;

  for (int tile = blockIdx.x; tile < tg.ntiles; tile += gridDim.x) {
    const int tzt = tile % tg.tz_tiles;
    const int rest = tile / tg.tz_tiles;
    const int tyt = rest % tg.ty_tiles;
    const int ch = rest / tg.ty_tiles;
    const int32_t y = tyt * kTY + ty, z = tzt * kTZ + tz;
    const int32_t xs = tg.x0 + ch * tg.xc;
    const int32_t xe = min(xs + tg.xc, tg.x1);
    // the halo slot this thread fills (64 along Y, 16 along Z)
    bool halo_cell = true;
    int hy = 0, hz = 0, sy_ = 0, sz_ = 0;
    if (threadIdx.x < 2 * kTZ) {
      const int side = threadIdx.x / kTZ;
      hy = tyt * kTY + (side ? kTY : -1);
      hz = z;
      sy_ = side ? kTY + 1 : 0;
      sz_ = tz + 1;
    } else if (threadIdx.x < 2 * kTZ + 2 * kTY) {
      const int k = threadIdx.x - 2 * kTZ;
      const int side = k / kTY;
      hy = tyt * kTY + (k % kTY);
      hz = tzt * kTZ + (side ? kTZ : -1);
      sy_ = (k % kTY) + 1;
      sz_ = side ? kTZ + 1 : 0;
    } else {
      halo_cell = false;
    }
    auto issue_plane = [&](int32_t x) {
      const int b = slot(x);
      issue(b, x, y, z, ty + 1, tz + 1);
      if (halo_cell) issue(b, x, hy, hz, sy_, sz_);
      cp_async_commit();
    };
    // g of plane x (tile + halo) from its raw buffer into g buffer x & 1
    auto convert = [&](int32_t x, double (&gcen)[3], double (&pcen)[3]) {
      const int b = slot(x);
      const int gb2 = x & 1;
      G(b, ty + 1, tz + 1, gcen, pcen);
#pragma unroll
      for (int q = 0; q < 3; ++q) gbuf[gb2][q][ty + 1][tz + 1] = gcen[q];
      if (halo_cell) {
        double hg[3], tmp[3];
        G(b, sy_, sz_, hg, tmp);
#pragma unroll
        for (int q = 0; q < 3; ++q) gbuf[gb2][q][sy_][sz_] = hg[q];
      }
    };

    double gm[3], gc[3], gn[3], pc[3], pn[3], tmp[3];
    __syncthreads();  // the previous tile is done with every buffer
    // planes xs - 1 .. xs + kStages - 2 in flight; wait for the first two
    for (int k = 0; k < kStages; ++k) {
      if (xs - 1 + k <= xe) issue_plane(xs - 1 + k);
      else cp_async_commit();
    }
    cp_async_wait<kStages - 2>();
    __syncthreads();
    G(slot(xs - 1), ty + 1, tz + 1, gm, tmp);
    convert(xs, gc, pc);
    __syncthreads();  // raw slot of plane xs - 1 is free again
    if (xs + kStages - 1 <= xe) issue_plane(xs + kStages - 1);
    else cp_async_commit();
    for (int32_t x = xs; x < xe; ++x) {
      const int64_t i = (int64_t)x * sX + (int64_t)y * sY + z;
      // this plane's coefficients (and r^): plain loads, consumed after the
      // barrier and the conversion of plane x + 1
      double cf[6];
      if (kTrans) {
        // the neighbour's coefficient across its back face
        bool ok;
        const int32_t xm = wrap(x - 1, tg.X, tg.px, ok);
        cf[0] = ok ? a[(int64_t)2 * n + xm * sX + (int64_t)y * sY + z] : 0.0;
        const int32_t xp = wrap(x + 1, tg.X, tg.px, ok);
        cf[1] = ok ? a[(int64_t)1 * n + xp * sX + (int64_t)y * sY + z] : 0.0;
        const int32_t ym = wrap(y - 1, tg.Y, tg.py, ok);
        cf[2] = ok ? a[(int64_t)4 * n + x * sX + (int64_t)ym * sY + z] : 0.0;
        const int32_t yp = wrap(y + 1, tg.Y, tg.py, ok);
        cf[3] = ok ? a[(int64_t)3 * n + x * sX + (int64_t)yp * sY + z] : 0.0;
        const int32_t zm = wrap(z - 1, tg.Z, tg.pz, ok);
        cf[4] = ok ? a[(int64_t)6 * n + x * sX + (int64_t)y * sY + zm] : 0.0;
        const int32_t zp = wrap(z + 1, tg.Z, tg.pz, ok);
        cf[5] = ok ? a[(int64_t)5 * n + x * sX + (int64_t)y * sY + zp] : 0.0;
      } else {
#pragma unroll
        for (int f = 0; f < 6; ++f) cf[f] = a[(int64_t)(1 + f) * n + i];
      }
      const double aii = a[i];
      double rh[3];
#pragma unroll
      for (int q = 0; q < 3; ++q)
        rh[q] = (MODE == 0 && q < nc && act[q]) ? w.rhat[q * n + i]
                : (kX && !kZ && q < nc && act[q]) ? bin[q * n + i]
                                                  : 0.0;
      cp_async_wait<kStages - 2>();  // my copies of plane x + 1 have landed
      __syncthreads();  // everyone's have; g of plane x is complete
      convert(x + 1, gn, pn);
      if (x + kStages <= xe) issue_plane(x + kStages);
      else cp_async_commit();
      const int gb = x & 1;
      if (kZ) {
        const double di = w.dinv[i];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q >= nc || !act[q]) continue;
          const double off = cf[0] * gm[q] + cf[1] * gn[q] +
                             cf[2] * gbuf[gb][q][ty][tz + 1] +
                             cf[3] * gbuf[gb][q][ty + 2][tz + 1] +
                             cf[4] * gbuf[gb][q][ty + 1][tz] +
                             cf[5] * gbuf[gb][q][ty + 1][tz + 2];
          xout[q * n + i] += gc[q] - di * off;
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (kZ || q >= nc || !act[q]) continue;
        const double yv = aii * gc[q] + cf[0] * gm[q] + cf[1] * gn[q] +
                          cf[2] * gbuf[gb][q][ty][tz + 1] +
                          cf[3] * gbuf[gb][q][ty + 2][tz + 1] +
                          cf[4] * gbuf[gb][q][ty + 1][tz] +
                          cf[5] * gbuf[gb][q][ty + 1][tz + 2];
        const int64_t o = q * n + i;
        if (MODE == 0) {
          vout[o] = yv;
          pout[o] = pc[q];
          acc[q] += rh[q] * yv;
        } else if (MODE == 1) {
          vout[o] = yv;
          acc[3 * q] += pc[q] * pc[q];
          acc[3 * q + 1] += yv * yv;
          acc[3 * q + 2] += yv * pc[q];
        } else {
          const double rr = rh[q] - yv;  // b - A x
          if (MODE == 2) {
            w.r[o] = rr;
            w.rhat[o] = rr;
            acc[3 + q] += rh[q] * rh[q];
          }
          acc[q] += rr * rr;
        }
      }
      if (MODE == 2) w.dinv[i] = pc_on ? 1.0 / aii : 1.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        gm[q] = gc[q];
        gc[q] = gn[q];
        pc[q] = pn[q];
      }
    }
    cp_async_wait_all();
  }
  if (kZ) return;
  double tot[K];
  if (!grid_reduce<K>(acc, partials, counter, tot)) return;
  if (MODE == 3) {
    for (int q = 0; q < nc; ++q) st->c[q].true_res = sqrt(tot[q]);
    return;
  }
  if (MODE == 2) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (act[q] && c.bnorm == 0.0) {
        // fresh solve: |b| and the absolute tolerance (k_bi_bnorm)
        c.bnorm = sqrt(tot[3 + q]);
        c.tol_abs = c.tol * c.bnorm;
        if (c.bnorm == 0.0) {
          c.zero_rhs = 1;
          c.done = 1;
          c.converged = 1;
        }
      }
      if (act[q] && !c.done) {
        c.res = sqrt(tot[q]);
        if (c.res <= c.tol_abs) {
          c.converged = 1;
          c.done = 1;
        } else {
          c.rho = c.alpha = c.omega = 1.0;
          c.iter = 1;
          c.rho_new = tot[q];
          if (fabs(c.rho_new) < DBL_MIN || fabs(c.omega) < DBL_MIN) {
            c.fail = 1;
            c.done = 1;
          } else {
            c.beta = (c.rho_new / c.rho) * (c.alpha / c.omega);
          }
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
    return;
  }
  if (MODE == 0) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (act[q]) {
        if (fabs(tot[q]) < DBL_MIN) {
          c.fail = 1;
          c.done = 1;
        } else {
          c.alpha = c.rho_new / tot[q];
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  } else {
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (!act[q]) continue;
      c.res = sqrt(tot[3 * q]);
      if (c.res <= c.tol_abs) {
        c.converged = 1;
        c.done = 1;
        c.pending = 1;
      } else if (tot[3 * q + 1] < DBL_MIN) {
        c.fail = 1;
        c.done = 1;
      } else {
        c.omega = tot[3 * q + 2] / tot[3 * q + 1];
      }
    }
  }
}

__global__ void __launch_bounds__(kBlock)
    k_bi_finish(double *__restrict__ x, int32_t n, Rng rg, const SolverState *st) {
  for (int q = 0; q < st->ncomp; ++q) {
    if (!st->c[q].zero_rhs) continue;
    RANGE_LOOP(i, rg) x[(int64_t)q * n + i] = 0.0;
  }
}

#include "bicg_nm.cuh"
#include "cg_tiled.cuh"

// Neumann-2 BiCGStab, behind a batch's last st pass: that iteration's x/r
// update (z += alpha p + omega s, r' = s - omega t with s = r - alpha v;
// converged-at-s components z += alpha p) and the residual test on r' --
// the pointwise part of the merged pass that would follow (168 B/cell for
// three components instead of the merged pass's stencil), so a batch sized
// by the hint ends converged.  The next merged pass, if the solve goes on,
// skips the update it would make (xr_applied) and repeats the same test.
__global__ void __launch_bounds__(kBlock)
    k_nm_xr(const double *__restrict__ r, const double *__restrict__ v,
            const double *__restrict__ p, const double *__restrict__ t,
            double *__restrict__ z, double *__restrict__ rout, int64_t n,
            Rng rg, SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  const int nc = st->ncomp;
  bool on[3], pend[3];
  double al[3], om[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    on[q] = q < nc && !st->c[q].done;
    pend[q] = q < nc && st->c[q].pending;
    al[q] = q < nc ? st->c[q].alpha : 0.0;
    om[q] = q < nc ? st->c[q].omega : 0.0;
  }
  double acc[3] = {0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int64_t j = q * n + i;
      if (on[q]) {
        const double sv = r[j] - al[q] * v[j];
        const double rn = sv - om[q] * t[j];
        rout[j] = rn;
        z[j] += al[q] * p[j] + om[q] * sv;
        acc[q] += rn * rn;
      } else if (pend[q]) {
        z[j] += al[q] * p[j];
      }
    }
  }
  double tot[3];
  if (!grid_reduce<3>(acc, partials, counter, tot)) return;
  int all = 1;
  for (int q = 0; q < nc; ++q) {
    CompState &c = st->c[q];
    if (on[q]) {
      // the merged pass's terminal decisions (bicg_nm.cuh epilogue)
      c.res = sqrt(tot[q]);
      if (c.res <= c.tol_abs) {
        c.converged = 1;
        c.done = 1;
      } else if (c.iter >= c.maxiter) {
        c.done = 1;
      } else if (c.brk_next) {
        c.fail = 1;
        c.done = 1;
      }
    }
    if (on[q] || pend[q]) c.xr_applied = 1;
    if (!c.done) all = 0;
  }
  st->all_done = all;
}

}  // namespace pf

// ===========================================================================
// host drivers

using namespace pf;

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

// PF_NO_SPECULATIVE=1: close a solve (finish, true residual) only after the
// poll that saw it converge (an A/B switch for the speculative close)
static bool speculative_close() {
  static const bool on = [] {
    const char *e = getenv("PF_NO_SPECULATIVE");
    return !(e && e[0] == '1');
  }();
  return on;
}

static int read_state(const Plan &pl, SolverState *dev, SolverState *host,
                      cudaStream_t s) {
  return d2h(pl, host, dev, sizeof(SolverState), s);
}

namespace {

// iterations to launch before the next host poll
int next_batch(int done_iters, int hint) {
  // PF_MAX_BATCH caps the iterations in flight between host polls (the
  // in-process slab tests: several slabs' launch queues share one context,
  // and a host thread blocked on a full queue must not starve a peer slab)
  static const int cap = [] {
    const char *e = getenv("PF_MAX_BATCH");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 64;
  }();
  int b = std::max(std::min(4, cap), std::min(cap, done_iters / 2));
  if (hint > done_iters) b = std::max(2, std::min(b, hint - done_iters));
  return b;
}

bool tile_geo_dim(const Plan &pl, int dim, TileGeo &tg);

// Pressure CG variant (k_cg1_*): 0 the classic loop (three fused reductions
// per iteration), 1 Chronopoulos-Gear with one reduction per iteration (the
// residual norm rides with r.z and z.w, so convergence is seen one
// preconditioner application late), 2 the same recurrence with the norm
// reduced in the update pass (two reductions, no extra application).  Every
// reduction is a cross-rank synchronisation on slab plans, which default to
// 2 (measured: the warm-started solves converge in one or two iterations,
// where variant 1's extra application outweighs the synchronisation it
// saves).  PF_CG_VARIANT=classic|single|split overrides; non-classic on one
// device is a test setting.
int cg_variant(const Plan &pl) {
  static const int env = [] {
    const char *e = getenv("PF_CG_VARIANT");
    if (!e) return -1;
    if (!strcmp(e, "classic")) return 0;
    if (!strcmp(e, "single")) return 1;
    if (!strcmp(e, "split")) return 2;
    return -1;
  }();
  return env >= 0 ? env : pl.slab ? 2 : 0;
}
bool cg_single(const Plan &pl) { return cg_variant(pl) != 0; }

// The fused direction update + SpMV on tiles (cg_tiled.cuh) applies on
// single-device 3D boxes whose level-0 face form is laid out as the box
// (PF_NO_TILED_CG=1: the per-cell gather SpMV and a separate update)
bool cg_tiled(const Plan &pl, const MgHierarchy *mg, TileGeo &tg) {
  static const bool off = getenv("PF_NO_TILED_CG") != nullptr;
  if (off || pl.slab || cg_single(pl) || !mg ||
      !tile_geo_dim(pl, pl.d.dim, tg))
    return false;
  const MgLevel &L = mg->lv[0];
  if (!(L.sx == tg.X && L.sy == tg.Y && L.sz == tg.Z && L.px == tg.px &&
        L.pz == tg.pz && !tg.py))
    return false;
  // X chunks for kCgMinB resident CTAs per SM (as tile_geo does for two)
  const int32_t nx = tg.x1 - tg.x0;
  const int64_t R = (int64_t)kCgMinB * pl.num_sms;
  const int64_t ncols = (int64_t)tg.ty_tiles * tg.tz_tiles;
  int64_t best = -1;
  for (int32_t xc = 1; xc <= std::max(1, nx); ++xc) {
    const int64_t tiles = ncols * ((nx + xc - 1) / xc);
    const int64_t cost = (tiles + R - 1) / R * (xc + 2);
    if (best < 0 || cost <= best) {
      best = cost;
      tg.xc = xc;
    }
  }
  tg.chunks = (nx + tg.xc - 1) / tg.xc;
  tg.ntiles = tg.ty_tiles * tg.tz_tiles * tg.chunks;
  return true;
}

template <int MODE>
void launch_cg_tiled(const TileGeo &tg, const Plan &pl, const MgLevel &L,
                     const double *z, double *p0, double *p1, double *q,
                     SolverState *st, Workspace &w, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_cg_tiled<MODE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kCgTileSmem);
  });
  count_launch();
  k_cg_tiled<MODE><<<std::min(tg.ntiles, std::min(pl.red_blocks,
                                                  kCgMinB * pl.num_sms)),
                     kTileThreads, kCgTileSmem, s>>>(
      tg, L, z, p0, p1, q, st, w.partials, w.counters, plan_range(pl));
}
void launch_cg_spmv_pt(const TileGeo &tg, const Plan &pl, const MgLevel &L,
                       const double *z, double *p0, double *p1, double *q,
                       SolverState *st, Workspace &w, cudaStream_t s) {
  launch_cg_tiled<0>(tg, pl, L, z, p0, p1, q, st, w, s);
}

// one multigrid-preconditioned CG iteration on workspace buffers only
// ---------------------------------------------------------------------------
// Single-reduction CG (Chronopoulos & Gear 1989): the reference's iterates
// (S/linalg.py:136-170) in exact arithmetic, with w = K z carried alongside
// so that the next step length follows from sums of one pass:
//
//   p = (z - zbar) + beta p      s = w + beta s   (= K p by linearity)
//   x += alpha p                 r -= alpha s
//   z = M r                      w = K z
//   gamma = r.(z - zbar)         delta = (z - zbar).w
//   beta = gamma / gamma_old     alpha = gamma / (delta - beta gamma / alpha_old)
//
// (z - zbar).w uses K 1 = 0 (face form, any walls): K (z - zbar) = K z.  The
// residual norm of the update rides in the same reduction, so convergence
// is seen one preconditioner application late; x is already the converged
// iterate then (the count reported is the reference's).

__device__ __forceinline__ void cg1_fail(SolverState *st) {
  CompState &c = st->c[0];
  c.fail = 1;
  c.done = 1;
  st->all_done = 1;
}

// w = K z and the six sums: r.r, sum z, r.z, sum r, z.w, sum w.  check: the
// residual test of the update before this pass happens here (variant 1);
// otherwise the update pass made it (variant 2)
__global__ void __launch_bounds__(kBlock)
    k_cg1_spmv(MgLevel L, Rng rg, const double *__restrict__ z,
               const double *__restrict__ r, double *__restrict__ w,
               int initial, int check, SolverState *st, double *partials,
               unsigned *counter) {
  if (st->all_done) return;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  RANGE_LOOP(i, rg) {
    const Cell3 c = decode(L, i);
    const double wi = kx(nbhd(L, c), i, z);
    const double zi = z[i], ri = r[i];
    w[i] = wi;
    acc[0] += ri * ri;
    acc[1] += zi;
    acc[2] += ri * zi;
    acc[3] += ri;
    acc[4] += zi * wi;
    acc[5] += wi;
  }
  double tot[6];
  if (!grid_reduce<6>(acc, partials, counter, tot)) return;
  CompState &c = st->c[0];
  if (!initial && check) {
    // the update before this pass was iteration c.iter + 1
    c.iter += 1;
    c.res = sqrt(tot[0]);
    if (c.res <= c.tol_abs) {
      c.converged = 1;
      c.done = 1;
      c.project_x = st->zero_mean;  // xmean: k_cg1_xmean in the close
      st->all_done = 1;
      return;
    }
    if (c.iter >= c.maxiter) {
      c.done = 1;
      st->all_done = 1;
      return;
    }
  }
  c.zbar = st->zero_mean ? tot[1] / rg.ng : 0.0;
  const double g = tot[2] - c.zbar * tot[3];
  const double d = tot[4] - c.zbar * tot[5];
  if (initial) {
    if (!pf::finite(d) || fabs(d) < DBL_MIN) return cg1_fail(st);
    c.rz = g;
    c.beta = 0.0;
    c.alpha = g / d;
    return;
  }
  if (!pf::finite(g) || c.rz == 0.0) return cg1_fail(st);
  const double beta = g / c.rz;
  const double pap = d - beta * g / c.alpha;  // p.K p of the next direction
  if (!pf::finite(pap) || fabs(pap) < DBL_MIN) return cg1_fail(st);
  c.beta = beta;
  c.rz = g;
  c.alpha = g / pap;
}

// p = (z - zbar) + beta p; s = w + beta s; x += alpha p; r -= alpha s (the
// first iteration reads no p / s).  kCheck (variant 2): |r| and sum x of
// the update, the residual test and the x mean of the projection here
template <bool kCheck>
__global__ void __launch_bounds__(kBlock)
    k_cg1_update(const double *__restrict__ z, const double *__restrict__ w,
                 double *__restrict__ p, double *__restrict__ sv,
                 double *__restrict__ x, double *__restrict__ r, Rng rg,
                 SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  const CompState &cs = st->c[0];
  const bool first = cs.iter == 0;
  const double beta = cs.beta, alpha = cs.alpha, zbar = cs.zbar;
  double acc[2] = {0.0, 0.0};
  RANGE_LOOP(i, rg) {
    double pi = z[i] - zbar, si = w[i];
    if (!first) {
      pi += beta * p[i];
      si += beta * sv[i];
    }
    p[i] = pi;
    sv[i] = si;
    const double xi = x[i] + alpha * pi, ri = r[i] - alpha * si;
    x[i] = xi;
    r[i] = ri;
    if (kCheck) {
      acc[0] += ri * ri;
      acc[1] += xi;
    }
  }
  if (!kCheck) return;
  double tot[2];
  if (!grid_reduce<2>(acc, partials, counter, tot)) return;
  CompState &c = st->c[0];
  c.iter += 1;
  c.res = sqrt(tot[0]);
  if (c.res <= c.tol_abs) {
    c.converged = 1;
    c.done = 1;
    c.project_x = st->zero_mean;
    c.xmean = st->zero_mean ? tot[1] / rg.ng : 0.0;
    st->all_done = 1;
  } else if (c.iter >= c.maxiter) {
    c.done = 1;
    st->all_done = 1;
  }
}

// mean of the converged x for the zero-mean projection (variant 1; the
// others get it from their update pass's reduction)
__global__ void __launch_bounds__(kBlock)
    k_cg1_xmean(const double *__restrict__ x, Rng rg, SolverState *st,
                double *partials, unsigned *counter) {
  if (!st->c[0].project_x) return;
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) acc[0] += x[i];
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot))
    st->c[0].xmean = tot[0] / rg.ng;
}

void mg_iteration(const Plan &pl, Workspace &w, SolverState *st,
                  const MgHierarchy *mg, double *x, cudaStream_t s) {
  const int32_t n = (int32_t)pl.d.n;
  double *r = w.vecs, *p = w.vecs + n, *q = w.vecs + 2 * (int64_t)n;
  double *z = w.vecs + 4 * (int64_t)n;
  const int ge = grid_for(pl.i1 - pl.i0), gr = std::min(ge, pl.red_blocks);
  const Rng rg = plan_range(pl);
  if (const int var = cg_variant(pl)) {
    double *wv = w.vecs + 7 * (int64_t)n;
    if (var == 2)
      launch(k_cg1_update<true>, gr, kBlock, s, (const double *)z,
             (const double *)wv, p, q, x, r, rg, st, w.partials, w.counters);
    else
      launch(k_cg1_update<false>, ge, kBlock, s, (const double *)z,
             (const double *)wv, p, q, x, r, rg, st, w.partials, w.counters);
    const CgFuse closes{nullptr, nullptr, nullptr, 0, 1};
    mg_apply(*mg, r, z, s, &st->all_done, nullptr, &closes, pl.red_blocks,
             &pl);
    halo(pl, s, {{z, 1}});
    launch(k_cg1_spmv, gr, kBlock, s, mg->lv[0], rg, (const double *)z,
           (const double *)r, wv, 0, var == 1 ? 1 : 0, st, w.partials,
           w.counters);
    return;
  }
  TileGeo tg;
  if (cg_tiled(pl, mg, tg)) {
    double *p1 = w.vecs + 6 * (int64_t)n;
    launch_cg_spmv_pt(tg, pl, mg->lv[0], z, p, p1, q, st, w, s);
    launch(k_cg_update_pt, gr, kBlock, s, (const double *)p,
           (const double *)p1, (const double *)q, x, r, rg, st, w.partials,
           w.counters);
    const CgFuse fuse{st, w.partials, w.counters, 0};
    mg_apply(*mg, r, z, s, &st->all_done, nullptr, &fuse, pl.red_blocks, &pl);
    return;
  }
  halo(pl, s, {{p, 1}});
  launch(k_cg_spmv_faces, gr, kBlock, s, mg->lv[0], rg, (const double *)p, q, st,
         w.partials, w.counters);
  launch(k_cg_update, gr, kBlock, s, (const double *)nullptr,
         (const double *)p, (const double *)q, x, r, rg, st, w.partials,
         w.counters);
  // the V-cycle's last smoothing pass also forms the z-sums and beta
  const CgFuse fuse{st, w.partials, w.counters, 0};
  mg_apply(*mg, r, z, s, &st->all_done, nullptr, &fuse, pl.red_blocks, &pl);
  launch(k_cg_pupdate, ge, kBlock, s, (const double *)nullptr,
         (const double *)r, (const double *)z, p, rg, st);
}

// r = bp - K x on the multigrid level-0 face form
__global__ void __launch_bounds__(kBlock)
    k_cg_resid_faces(MgLevel L, Rng rg, const double *__restrict__ bp,
                     const double *__restrict__ x, double *__restrict__ r,
                     SolverState *st, double *partials, unsigned *counter) {
  if (st->all_done) return;
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) {
    const Cell3 c = decode(L, i);
    const double ri = bp[i] - kx(nbhd(L, c), i, x);
    r[i] = ri;
    acc[0] += ri;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot))
    st->c[0].rmean = st->zero_mean ? tot[0] / rg.ng : 0.0;
}

// |bp - K x| on the face form (the true-residual verification of the
// preconditioned pressure CG, S/linalg.py:236-239): 40 B/cell instead of the
// 72 of the (2d+1)-row stencil
__global__ void __launch_bounds__(kBlock)
    k_cg_true_res_faces(MgLevel L, Rng rg, const double *__restrict__ bp,
                        const double *__restrict__ x, SolverState *st,
                        double *partials, unsigned *counter) {
  double acc[1] = {0.0};
  RANGE_LOOP(i, rg) {
    const Cell3 c = decode(L, i);
    const double ri = bp[i] - kx(nbhd(L, c), i, x);
    acc[0] += ri * ri;
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot))
    st->c[0].true_res = sqrt(tot[0]);
}


constexpr int kGraphIters = 4;  // MG-PCG iterations per graph launch

// Graph of kGraphIters iterations, cached on the plan for its buffers.
int mg_graph(const Plan &pl, Workspace &w, SolverState *st,
             const MgHierarchy *mg, double *x, cudaGraphExec_t *out,
             unsigned long long *nkern) {
  GraphCache &gc = pl.graph;
  const void *key[3] = {w.vecs, mg->lv[0].wx, x};
  if (gc.exec && gc.key[0] == key[0] && gc.key[1] == key[1] &&
      gc.key[2] == key[2]) {
    *out = gc.exec;
    *nkern = gc.nkern;
    return PF_OK;
  }
  if (gc.exec) {
    cudaGraphExecDestroy(gc.exec);
    gc.exec = nullptr;
  }
  if (!gc.cap) PF_CUDA(cudaStreamCreateWithFlags(&gc.cap, cudaStreamNonBlocking));
  unsigned long long captured = 0;
  g_capture_count = &captured;  // captured, not launched
  PF_CUDA(cudaStreamBeginCapture(gc.cap, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < kGraphIters; ++k) mg_iteration(pl, w, st, mg, x, gc.cap);
  cudaGraph_t graph;
  cudaError_t ec = cudaStreamEndCapture(gc.cap, &graph);
  g_capture_count = nullptr;
  PF_CUDA(ec);
  gc.nkern = captured;
  cudaError_t e = cudaGraphInstantiate(&gc.exec, graph, 0);
  cudaGraphDestroy(graph);
  PF_CUDA(e);
  for (int j = 0; j < 3; ++j) gc.key[j] = key[j];
  *out = gc.exec;
  *nkern = gc.nkern;
  return PF_OK;
}

template <class V>
int cg_core_mg(const Plan &pl, const V &v, Workspace &w, SolverState *st,
               SolverState &hs, const double *a, const double *bp, double *x,
               double tol, int maxiter, int zero_mean, const MgHierarchy *mg,
               cudaStream_t s, double *xout) {
  // x is the workspace copy of the warm start (the graph's buffers are all
  // workspace-resident); xout the caller's solution buffer
  const int32_t n = v.n;
  double *r = w.vecs, *p = w.vecs + n;
  double *z = w.vecs + 4 * (int64_t)n;
  const int *done = &st->all_done;
  const int ge = grid_for(pl.i1 - pl.i0), gr = std::min(ge, pl.red_blocks);
  const Rng rg = plan_range(pl);
  (void)a;
  launch(k_cg_reset, 1, 1, s, st, maxiter, 2, zero_mean, tol, 0);
  halo(pl, s, {{x, 1}});
  TileGeo tgr;
  if (cg_tiled(pl, mg, tgr))
    launch_cg_tiled<1>(tgr, pl, mg->lv[0], x, const_cast<double *>(bp), nullptr,
                       r, st, w, s);
  else
    launch(k_cg_resid_faces, gr, kBlock, s, mg->lv[0], rg, bp,
           (const double *)x, r, st, w.partials, w.counters);
  launch(k_cg_rproj, gr, kBlock, s, (const double *)nullptr, r, rg, st,
         w.partials, w.counters);
  const bool single = cg_single(pl);
  const CgFuse fuse{st, w.partials, w.counters, 1};
  const CgFuse closes{nullptr, nullptr, nullptr, 0, 1};  // k_cg1_spmv follows
  int rc = mg_apply(*mg, r, z, s, done, nullptr, single ? &closes : &fuse,
                    pl.red_blocks, &pl);
  if (rc) return rc;
  if (single) {
    // w0 = K z0 and the first step length (the update forms p0 = z0 - zbar)
    halo(pl, s, {{z, 1}});
    launch(k_cg1_spmv, gr, kBlock, s, mg->lv[0], rg, (const double *)z,
           (const double *)r, w.vecs + 7 * (int64_t)n, 1, 0, st, w.partials,
           w.counters);
  }
  // the tiled iteration forms the first direction itself (p = z - zbar)
  TileGeo tgc;
  if (!single && !cg_tiled(pl, mg, tgc))
    launch(k_cg_pinit, ge, kBlock, s, (const double *)nullptr, r,
           (const double *)z, p, rg, st);
  PF_LAUNCH_CHECK("mg-cg setup");
  // PF_NO_GRAPHS=1: launch the iterations directly (the in-process slab
  // tests: instantiating a graph may wait for the whole device while other
  // slabs' kernels spin on this one)
  static const bool no_graphs = [] {
    const char *e = getenv("PF_NO_GRAPHS");
    return e && e[0] == '1';
  }();
  cudaGraphExec_t exec = nullptr;
  unsigned long long nk = 0;
  if (!no_graphs) {
    rc = mg_graph(pl, w, st, mg, x, &exec, &nk);
    if (rc) return rc;
  }
  auto close = [&]() {
    if (cg_variant(pl) == 1)
      launch(k_cg1_xmean, gr, kBlock, s, (const double *)x, rg, st,
             w.partials, w.counters);
    launch(k_cg_finish, ge, kBlock, s, x, rg, st);
    PF_CUDA(cudaMemcpyAsync(xout, x, sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, s));
    halo(pl, s, {{xout, 1}});
    TileGeo tgv;
    if (cg_tiled(pl, mg, tgv))
      launch_cg_tiled<2>(tgv, pl, mg->lv[0], xout, const_cast<double *>(bp),
                         nullptr, nullptr, st, w, s);
    else
      launch(k_cg_true_res_faces, gr, kBlock, s, mg->lv[0], rg, bp,
             (const double *)xout, st, w.partials, w.counters);
    PF_LAUNCH_CHECK("mg-cg close");
    return PF_OK;
  };
  // the first batch goes out without a poll (its kernels return at once
  // when the setup already converged): one host round trip per batch
  int launched = 0;
  for (;;) {
    if (launched >= maxiter) break;  // maxiter <= 0: no iteration at all
    int b = std::min(next_batch(launched, 0), maxiter - launched);
    b = std::max(1, (b + kGraphIters - 1) / kGraphIters);
    for (int k = 0; k < b; ++k) {
      if (exec) {
        PF_CUDA(cudaGraphLaunch(exec, s));
        g_launches.fetch_add(nk, std::memory_order_relaxed);
      } else {
        for (int j = 0; j < kGraphIters; ++j)
          mg_iteration(pl, w, st, mg, x, s);
      }
    }
    launched += b * kGraphIters;
    const bool spec = speculative_close();
    // speculative close behind the batch (idempotent until a batch
    // converges, and the loop stops at the first that does): the zero-mean
    // projection of x, the copy out and the true-residual verification, so
    // a solve whose first batch converges costs one host round trip
    if (spec) close();
    rc = read_state(pl, st, &hs, s);
    if (!rc) rc = comm_check(pl, s);
    if (rc) return rc;
    if (hs.all_done || launched >= maxiter) {
      if (spec) return PF_OK;
      break;
    }
  }
  close();
  return read_state(pl, st, &hs, s);
}

template <class V>
int cg_core(const Plan &pl, const V &v, Workspace &w, SolverState *st,
            SolverState &hs, const double *a, const double *bp, double *x,
            double tol, int maxiter, int precond, int zero_mean,
            const MgHierarchy *mg, cudaStream_t s) {
  const int32_t n = v.n;
  double *r = w.vecs, *p = w.vecs + n, *q = w.vecs + 2 * (int64_t)n;
  double *z = w.vecs + 4 * (int64_t)n;
  const int *done = &st->all_done;
  const int ge = grid_for(pl.i1 - pl.i0), gr = std::min(ge, pl.red_blocks);
  const Rng rg = plan_range(pl);
  if (precond == 2) {
    // the multigrid iteration runs from a CUDA graph whose buffers are all
    // workspace-resident: iterate on a copy of x, copy the solution back
    double *xw = w.vecs + 5 * (int64_t)n;
    PF_CUDA(cudaMemcpyAsync(xw, x, sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, s));
    // the close (projection, copy back, true residual) rides behind each
    // batch inside cg_core_mg; hs is read after it
    return cg_core_mg(pl, v, w, st, hs, a, bp, xw, tol, maxiter, zero_mean,
                      mg, s, x);
  }
  launch(k_cg_reset, 1, 1, s, st, maxiter, precond, zero_mean, tol, 0);
  halo(pl, s, {{x, 1}});
  launch(k_cg_resid<V>, gr, kBlock, s, v, a, bp, x, r, st, w.partials,
                                      w.counters);
  launch(k_cg_rproj, gr, kBlock, s, a, r, rg, st, w.partials, w.counters);
  (void)done;
  launch(k_cg_pinit, ge, kBlock, s, a, r, (const double *)z, p, rg, st);
  PF_LAUNCH_CHECK("cg setup");
  int launched = 0;
  for (;;) {
    if (launched >= maxiter) {  // maxiter <= 0: no iteration at all
      const int rc = read_state(pl, st, &hs, s);
      if (rc) return rc;
      break;
    }
    const int b = std::min(next_batch(launched, 0), maxiter - launched);
    for (int k = 0; k < b; ++k) {
      halo(pl, s, {{p, 1}});
      launch(k_cg_spmv<V>, gr, kBlock, s, v, a, p, q, st, w.partials,
             w.counters);
      launch(k_cg_update, gr, kBlock, s, a, p, q, x, r, rg, st, w.partials,
                                        w.counters);
      launch(k_cg_pupdate, ge, kBlock, s, a, r, (const double *)z, p, rg, st);
    }
    PF_LAUNCH_CHECK("cg iterations");
    launched += b;
    int rc = read_state(pl, st, &hs, s);
    if (!rc) rc = comm_check(pl, s);
    if (rc) return rc;
    if (hs.all_done || launched >= maxiter) break;
  }
  launch(k_cg_finish, ge, kBlock, s, x, rg, st);
  if (hs.c[0].converged && !hs.c[0].zero_rhs) {
    halo(pl, s, {{x, 1}});
    launch(k_true_res<V>, gr, kBlock, s, v, a, 0, 1, bp, x, st, w.partials,
                                        w.counters);
  }
  PF_LAUNCH_CHECK("cg finish");
  return read_state(pl, st, &hs, s);
}

}  // namespace

extern "C" int pf_cg_solve(const pf_plan *plan, const double *a,
                           const double *b, double b_scale, double *x,
                           int32_t has_x0,
                           double tol, int32_t maxiter, int32_t zero_mean,
                           int32_t precond, void *workspace,
                           void *mg_workspace,
                           pf_solver_report *report_host, void *stream) {
  if (!plan || !a || !b || !x || !workspace || !report_host || maxiter < 0 ||
      precond < 0 || precond > 2) {
    set_error("pf_cg_solve: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  MgHierarchy mg;
  if (precond == 2) {
    if (!pl.has_mg || !mg_workspace) {
      set_error("pf_cg_solve: multigrid preconditioner unavailable (needs a "
                "box plan and an MG workspace set up by pf_mg_setup)");
      return PF_ERR_UNSUPPORTED;
    }
    mg = pl.mg;
    mg_bind(mg, mg_workspace);
  }
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  SolverState *st = reinterpret_cast<SolverState *>(w.solver);
  cudaStream_t s = S(stream);
  const int32_t n = (int32_t)pl.d.n;
  double *bp = w.vecs + 3 * (int64_t)n;
  return dispatch(pl, [&](auto v) {
    using V = decltype(v);
    const int gr = std::min(grid_for(pl.i1 - pl.i0), pl.red_blocks);
    const Rng rg = plan_range(pl);
    SolverState hs;
    if (!has_x0) PF_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    launch(k_cg_reset, 1, 1, s, st, maxiter, precond, zero_mean, tol, 1);
    launch(k_cg_bsum, gr, kBlock, s, b, b_scale, rg, st, w.partials,
                                    w.counters);
    launch(k_cg_bproj, gr, kBlock, s, b, b_scale, bp, rg, st, w.partials,
                                     w.counters);
    PF_LAUNCH_CHECK("cg rhs");
    int rc = cg_core<V>(pl, v, w, st, hs, a, bp, x, tol, maxiter, precond,
                        zero_mean, &mg, s);
    if (rc) return rc;
    const CompState &c = hs.c[0];
    pf_solver_report rep;
    rep.fallback_used = 0;
    rep.breakdown = c.fail;
    if (c.zero_rhs) {
      rep.converged = 1;
      rep.iterations = 0;
      rep.residual = 0.0;
      *report_host = rep;
      return PF_OK;
    }
    bool ok = c.converged && c.true_res <= 10.0 * c.tol_abs;
    double res = c.converged ? c.true_res : c.res;
    int iters = c.iter;
    const double bnorm = c.bnorm;
    if (!ok && precond) {
      rep.fallback_used = 1;
      PF_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
      rc = cg_core<V>(pl, v, w, st, hs, a, bp, x, tol, 2 * maxiter, 0,
                      zero_mean, &mg, s);
      if (rc) return rc;
      const CompState &c2 = hs.c[0];
      iters += c2.iter;
      ok = c2.converged && c2.true_res <= 10.0 * c2.tol_abs;
      res = c2.converged ? c2.true_res : c2.res;
      rep.breakdown = c2.fail;
    }
    rep.converged = ok;
    rep.iterations = iters;
    rep.residual = bnorm > 0 ? res / bnorm : 0.0;
    *report_host = rep;
    return PF_OK;
  });
}

namespace {

template <bool kTrans, int MODE>
void launch_tiled(const TileGeo &tg, int grid, cudaStream_t s, const double *a,
                  const BiVecs &bv, int par, int64_t n, SolverState *st,
                  Workspace &w, const double *xin = nullptr,
                  const double *bin = nullptr, int nverify = 0,
                  int first = 0, double *xout = nullptr) {
  // 2 CTAs per SM (<= 128 registers, 2 x 71 KB of shared memory) measured
  // best on C4: pass pv 5.3 TB/s, pass st 4.3 TB/s (1 CTA: 3.8 / 2.9; 3 CTAs
  // with the 80-register cap: 3.5 / 3.2).  PF_TILE_MINB overrides.
  static const int minb = [] {
    const char *e = getenv("PF_TILE_MINB");
    return e ? atoi(e) : 2;
  }();
  auto go = [&](auto kernel) {
    // the shared-memory opt-in, once per kernel (instantiations share the
    // lambda's type, so the flag is keyed by the kernel's address)
    static std::mutex mu;
    static std::set<const void *> done;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (done.insert(reinterpret_cast<const void *>(kernel)).second)
        cudaFuncSetAttribute(kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TileLayout<MODE>::kBytes);
    }
    count_launch();
    kernel<<<grid, kTileThreads, TileLayout<MODE>::kBytes, s>>>(tg, a, bv, par, n, st,
                                                 w.partials, w.counters, xin,
                                                 bin, nverify, xout);
  };
  if (MODE == 0 && first) {
    if (minb >= 3)
      go(k_bi_tiled<kTrans, MODE, 3, true>);
    else if (minb == 2)
      go(k_bi_tiled<kTrans, MODE, 2, true>);
    else
      go(k_bi_tiled<kTrans, MODE, 1, true>);
  } else if (minb >= 3) {
    go(k_bi_tiled<kTrans, MODE, 3>);
  } else if (minb == 2) {
    go(k_bi_tiled<kTrans, MODE, 2>);
  } else {
    go(k_bi_tiled<kTrans, MODE, 1>);
  }
}

// tiled stencil passes apply to 3D boxes whose Y / Z extents are whole tiles
bool tile_geo_dim(const Plan &pl, int dim, TileGeo &tg);
template <class V>
bool tile_geo(const Plan &pl, const V &v, TileGeo &tg) {
  (void)v;
  return tile_geo_dim(pl, V::kDim, tg);
}
bool tile_geo_dim(const Plan &pl, int dim, TileGeo &tg) {
  if (dim != 3 || pl.d.topo != PF_TOPO_BOX) return false;
  if (getenv("PF_NO_TILED")) return false;
  tg.X = (int32_t)pl.d.box_shape[0];
  tg.Y = (int32_t)pl.d.box_shape[1];
  tg.Z = (int32_t)pl.d.box_shape[2];
  if (tg.Y % kTY || tg.Z % kTZ) return false;
  tg.px = pl.d.box_periodic[0];
  tg.py = pl.d.box_periodic[1];
  tg.pz = pl.d.box_periodic[2];
  const int64_t plane = (int64_t)tg.Y * tg.Z;
  tg.x0 = (int32_t)(pl.i0 / plane);
  tg.x1 = (int32_t)(pl.i1 / plane);
  tg.ty_tiles = tg.Y / kTY;
  tg.tz_tiles = tg.Z / kTZ;
  // X chunk length: tiles run in rounds of R resident CTAs (two per SM), a
  // tile of xc planes costs ~ xc + 2 plane steps (its two prologue planes),
  // so pick xc minimising rounds * (xc + 2).  C4 (192 columns x 256
  // planes, R = 296): xc = 86, 576 tiles in 2 full rounds, instead of the
  // 768 tiles of xc = 64 whose third round is 59 % full.  Small boxes get
  // short chunks and enough tiles to fill the GPU.
  const int32_t nx = tg.x1 - tg.x0;
  {
    static const int minb = [] {
      const char *e = getenv("PF_TILE_MINB");
      return e ? std::max(1, atoi(e)) : 2;
    }();
    const int64_t R = (int64_t)std::min(minb, 3) * pl.num_sms;
    const int64_t ncols = (int64_t)tg.ty_tiles * tg.tz_tiles;
    int64_t best = -1;
    tg.xc = 1;
    for (int32_t xc = 1; xc <= std::max(1, nx); ++xc) {
      const int64_t tiles = ncols * ((nx + xc - 1) / xc);
      const int64_t cost = (tiles + R - 1) / R * (xc + 2);
      if (best < 0 || cost <= best) {
        best = cost;
        tg.xc = xc;
      }
    }
    static const int force = [] {  // PF_TILE_XC: fixed chunk (experiments)
      const char *e = getenv("PF_TILE_XC");
      return e ? atoi(e) : 0;
    }();
    if (force > 0) tg.xc = std::min(force, std::max(1, nx));
  }
  tg.chunks = (nx + tg.xc - 1) / tg.xc;
  tg.ntiles = tg.ty_tiles * tg.tz_tiles * tg.chunks;
  return true;
}

constexpr int kPrecondNeumann2 = 3;

// tile geometry of the Neumann-2 passes: the tiled geometry with chunks
// costed at xc + 4 planes (two prologue planes per stencil stage), two
// CTAs per SM.  Slab plans also get the edge-pass geometry (`edge`: one
// chunk on the first and one on the last owned plane).
// resident CTAs per SM of the Neumann-2 passes (PF_NM_MINB: 1 or 2).  One
// CTA (up to 255 registers) measured best on C4: the 128-register cap of
// two CTAs spills (pv 766-830 us vs 868-1289 us)
inline int nm_minb() {
  static const int m = [] {
    const char *e = getenv("PF_NM_MINB");
    return e && atoi(e) == 2 ? 2 : 1;
  }();
  return m;
}

template <class V>
bool nm_geo(const Plan &pl, const V &v, TileGeo &tg, TileGeo *edge = nullptr) {
  if (getenv("PF_NO_NEUMANN")) return false;
  if (!tile_geo(pl, v, tg)) return false;
  if (tg.X < 4 && !pl.slab) return false;
  if (edge) {
    *edge = tg;
    const int32_t nxl = tg.x1 - tg.x0;
    edge->xc = std::max(1, nxl - 1);
    edge->chunks = nxl > 1 ? 2 : 1;
    edge->ntiles = tg.ty_tiles * tg.tz_tiles * edge->chunks;
  }
  const int32_t nx = tg.x1 - tg.x0;
  const int64_t R = nm_minb() * (int64_t)pl.num_sms;
  const int64_t ncols = (int64_t)tg.ty_tiles * tg.tz_tiles;
  int64_t best = -1;
  for (int32_t xc = 1; xc <= std::max(1, nx); ++xc) {
    const int64_t tiles = ncols * ((nx + xc - 1) / xc);
    const int64_t cost = (tiles + R - 1) / R * (xc + 4);
    if (best < 0 || cost <= best) {
      best = cost;
      tg.xc = xc;
    }
  }
  tg.chunks = (nx + tg.xc - 1) / tg.xc;
  tg.ntiles = tg.ty_tiles * tg.tz_tiles * tg.chunks;
  return true;
}

// rpar: which r buffer (bv.rb) the pass reads (MODE 1, 3); MODE 3 writes
// the other
template <bool kTrans, int MODE>
void launch_nm(const TileGeo &tg, int grid, cudaStream_t s, const double *a,
               const BiVecs &bv, int par, int64_t n, SolverState *st,
               Workspace &w, int first = 0, const double *zin = nullptr,
               double *xout = nullptr, const double *qghost = nullptr,
               double *qedge = nullptr, int rpar = 0) {
  NmArgs g{};
  const double *rin = bv.rb[0] ? bv.rb[rpar] : bv.r;
  for (int q = 0; q < 3; ++q) {
    const int64_t o = q * n;
    g.src[0][q] = (MODE == 2 ? zin : rin) + o;
    g.src[1][q] = (MODE == 0 || MODE == 3 ? bv.v[par] : bv.v[par ^ 1]) + o;
    g.src[2][q] = bv.p[par] + o;
    g.src[3][q] = bv.t + o;
    g.rout[q] = bv.rb[0] ? bv.rb[rpar ^ 1] + o : nullptr;
    g.zio[q] = bv.z ? bv.z + o : nullptr;
    g.rhat[q] = bv.rhat + o;
    g.out1[q] = (MODE == 2 ? xout : qedge ? qedge : bv.p[par ^ 1]) + o;
    g.out2[q] = (MODE == 0 || MODE == 3 ? bv.v[par ^ 1] : bv.t) + o;
    g.qghost[q] = qghost ? qghost + o : nullptr;
  }
  g.dinv = bv.dinv;
  for (int f = 0; f < 6; ++f) g.row[f] = a + (1 + (kTrans ? f ^ 1 : f)) * n;
  g.X = tg.X;
  g.Y = tg.Y;
  g.Z = tg.Z;
  g.px = tg.px;
  g.py = tg.py;
  g.pz = tg.pz;
  g.sX = tg.Y * tg.Z;
  const int edge = qedge != nullptr;
  auto go = [&](auto kernel) {
    static std::mutex mu;
    static std::set<const void *> done;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (done.insert(reinterpret_cast<const void *>(kernel)).second)
        cudaFuncSetAttribute(kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)nm_smem<kTrans>());
    }
    count_launch();
    kernel<<<grid, kTileThreads, nm_smem<kTrans>(), s>>>(tg, g, st, w.partials,
                                                         w.counters, edge);
  };
  if (nm_minb() == 1) {
    if constexpr (MODE == 0) {
      if (first) {
        go(k_bi_nm<kTrans, MODE, true, 1>);
        return;
      }
    }
    go(k_bi_nm<kTrans, MODE, false, 1>);
    return;
  }
  if constexpr (MODE == 0) {
    if (first) {
      go(k_bi_nm<kTrans, MODE, true>);
      return;
    }
  }
  go(k_bi_nm<kTrans, MODE, false>);
}

// One Neumann-2 BiCGStab iteration i (0-based): the pv pass (i = 0) or
// the merged pass (iteration i-1's x/r update + iteration i's pv), then
// the st pass; slab plans first run each stencil pass's edge planes and
// exchange them (Q).  r ping-pongs: iteration i reads rb[i & 1].
template <bool kTrans>
void nm_iteration(const Plan &pl, const TileGeo &tgn, const TileGeo &tge,
                  int ngrid, int egrid, cudaStream_t s, const double *a,
                  const BiVecs &bv, int i, int64_t n, int ncomp,
                  SolverState *st, Workspace &w, double *qg) {
  const int par = i & 1;
  if (i == 0) {
    halo(pl, s, {{bv.rb[0], ncomp}, {bv.p[par], ncomp}});
    if (qg) {
      launch_nm<kTrans, 0>(tge, egrid, s, a, bv, par, n, st, w, 1, nullptr,
                           nullptr, nullptr, qg);
      halo(pl, s, {{qg, ncomp}});
    }
    launch_nm<kTrans, 0>(tgn, ngrid, s, a, bv, par, n, st, w, 1, nullptr,
                         nullptr, qg);
  } else {
    const int rp = (i - 1) & 1;
    halo(pl, s, {{bv.rb[rp], ncomp}, {bv.p[par], ncomp}, {bv.t, ncomp}});
    if (qg) {
      launch_nm<kTrans, 3>(tge, egrid, s, a, bv, par, n, st, w, 0, nullptr,
                           nullptr, nullptr, qg, rp);
      halo(pl, s, {{qg, ncomp}});
    }
    launch_nm<kTrans, 3>(tgn, ngrid, s, a, bv, par, n, st, w, 0, nullptr,
                         nullptr, qg, nullptr, rp);
  }
  halo(pl, s, {{bv.v[par ^ 1], ncomp}, {bv.rb[par], ncomp}});
  if (qg) {
    launch_nm<kTrans, 1>(tge, egrid, s, a, bv, par, n, st, w, 0, nullptr,
                         nullptr, nullptr, qg, par);
    halo(pl, s, {{qg, ncomp}});
  }
  launch_nm<kTrans, 1>(tgn, ngrid, s, a, bv, par, n, st, w, 0, nullptr,
                       nullptr, qg, nullptr, par);
}

template <class V, bool kTrans>
int bi_core(const Plan &pl, const V &v, Workspace &w, SolverState *st,
            SolverState &hs, const double *a, const double *b, double *x,
            int ncomp, double tol, int maxiter, int precond, unsigned mask,
            int fresh, cudaStream_t s) {
  const int32_t n = v.n;
  const int64_t len = (int64_t)ncomp * n;
  BiVecs bv;
  double *base = w.vecs;
  bv.r = base;
  bv.rhat = base + len;
  bv.t = base + 2 * len;
  bv.p[0] = base + 3 * len;
  bv.p[1] = base + 4 * len;
  bv.v[0] = base + 5 * len;
  bv.v[1] = base + 6 * len;
  bv.dinv = base + 7 * len;
  const int ge = grid_for(pl.i1 - pl.i0), gr = std::min(ge, pl.red_blocks);
  const Rng rg = plan_range(pl);
  TileGeo tg, tgn;
  const bool tiled = tile_geo(pl, v, tg);
  const int tgrid = tiled ? std::min(tg.ntiles, pl.red_blocks) : 0;
  // Neumann-2 (PRECOND_NEUMANN2) runs fused on tiled boxes (slab plans
  // with the edge passes); on generic grids the request degrades to Jacobi
  TileGeo tge;
  const bool nm = precond == kPrecondNeumann2 && nm_geo(pl, v, tgn, &tge);
  if (precond == kPrecondNeumann2 && !nm) precond = 1;
  const int ngrid = nm ? std::min(tgn.ntiles, nm_minb() * pl.num_sms) : 0;
  const int egrid = nm ? std::min(tge.ntiles, nm_minb() * pl.num_sms) : 0;
  double *z = base + 8 * len;  // the preconditioned iterate (nm)
  double *qg = pl.slab ? base + 9 * len : nullptr;  // slab edge stage 1
  if (nm) {
    bv.rb[0] = bv.r;
    bv.rb[1] = base + 10 * len;
    bv.z = z;
  }
  launch(k_bi_reset, 1, 1, s, st, ncomp, maxiter, precond, tol, fresh, mask);
  // init / verification on the tiled passes, or the per-cell gather kernels
  // (PF_TILED_SETUP=0)
  static const bool tsetup = [] {
    const char *e = getenv("PF_TILED_SETUP");
    return !(e && atoi(e) == 0);
  }();
  const bool tinit = tiled && tsetup;
  // the tiled init pass forms |b| itself
  if (fresh && !tinit)
    launch(k_bi_bnorm, gr, kBlock, s, b, n, rg, st, w.partials, w.counters);
  halo(pl, s, {{x, ncomp}});
  if (tinit)
    launch_tiled<kTrans, 2>(tg, tgrid, s, a, bv, 0, (int64_t)n, st, w, x, b, 0);
  else
    launch(k_bi_init<V, kTrans>, gr, kBlock, s, v, a, b, x, bv, st,
           w.partials, w.counters);
  // slab plans: the stencil passes gather r, p, v and 1 / A_jj of the
  // neighbours (v[0] = 0 and dinv are exchanged once here)
  halo(pl, s, {{bv.v[0], ncomp}, {bv.dinv, 1}});
  PF_LAUNCH_CHECK("bicgstab setup");
  // the first batch goes out without a poll (its kernels return at once
  // when the setup already converged)
  int launched = 0;
  for (;;) {
    if (launched >= maxiter) {  // maxiter <= 0: no iteration at all
      const int rc = read_state(pl, st, &hs, s);
      if (rc) return rc;
      break;
    }
    // first batch: the previous solve's lock-step count on this plan and
    // direction (time steps change slowly), so a typical solve polls once
    static const bool use_hint = getenv("PF_NO_HINT") == nullptr;
    const int hint = use_hint ? pl.bi_hint[kTrans ? 1 : 0] : 0;
    const int first = hint > 0 ? std::min(std::max(2, hint), 64) : 2;
    const int bsz = std::min(launched == 0 ? first
                             : launched < 4 ? 2
                                            : next_batch(launched, 0),
                             maxiter - launched);
    for (int k = 0; k < bsz; ++k) {
      const int i = launched + k, par = i & 1;
      if (nm) {
        nm_iteration<kTrans>(pl, tgn, tge, ngrid, egrid, s, a, bv, i,
                             (int64_t)n, ncomp, st, w, qg);
        continue;
      }
      halo(pl, s, {{bv.r, ncomp}, {bv.p[par], ncomp}});
      if (tiled)
        launch_tiled<kTrans, 0>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w,
                                nullptr, nullptr, 0, i == 0);
      else
        launch(k_bi_pv<V, kTrans>, gr, kBlock, s, v, a, bv, par, st,
               w.partials, w.counters);
      halo(pl, s, {{bv.v[par ^ 1], ncomp}});
      if (tiled)
        launch_tiled<kTrans, 1>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w);
      else
        launch(k_bi_st<V, kTrans>, gr, kBlock, s, v, a, bv, par, st,
               w.partials, w.counters);
      launch(k_bi_xr<false>, gr, kBlock, s, a, bv, par, x, n, rg, st,
             w.partials, w.counters, 0);
    }
    PF_LAUNCH_CHECK("bicgstab iterations");
    launched += bsz;
    if (nm) {
      // the last iteration's x/r update and residual test (k_nm_xr), then
      // the speculative close x = x0 + M^-1 z (a one-stage stencil on the
      // single-halo tiled pass, which skips itself unless the solve ended)
      const int par = launched & 1, rp = (launched - 1) & 1;
      launch(k_nm_xr, gr, kBlock, s, (const double *)bv.rb[rp],
             (const double *)bv.v[par], (const double *)bv.p[par],
             (const double *)bv.t, z, bv.rb[par], (int64_t)n, rg, st,
             w.partials, w.counters);
      if (speculative_close()) {
        halo(pl, s, {{z, ncomp}});
        launch_tiled<kTrans, 4>(tg, tgrid, s, a, bv, 0, (int64_t)n, st, w, z,
                                nullptr, 1, 0, x);
      }
    }
    if (speculative_close()) {
      // speculative close: the finish and the true-residual verification
      // go out behind the batch (both idempotent), so a batch sized right
      // by the hint costs one host round trip for the whole solve
      launch(k_bi_finish, ge, kBlock, s, x, n, rg, st);
      halo(pl, s, {{x, ncomp}});
      if (tinit)
        launch_tiled<kTrans, 3>(tg, tgrid, s, a, bv, 0, (int64_t)n, st, w, x,
                                b, ncomp);
      else
        launch(k_true_res<V>, gr, kBlock, s, v, a, kTrans ? 1 : 0, ncomp, b,
               x, st, w.partials, w.counters);
      PF_LAUNCH_CHECK("bicgstab finish");
    }
    int rc = read_state(pl, st, &hs, s);
    if (!rc) rc = comm_check(pl, s);
    if (rc) return rc;
    if (hs.all_done || launched >= maxiter) break;
  }
  {
    int lock = 0;  // lock-step iterations this solve needed
    for (int q = 0; q < ncomp; ++q) lock = std::max(lock, (int)hs.c[q].iter);
    pl.bi_hint[kTrans ? 1 : 0] = lock;
  }
  // the speculative close already ran behind the last batch (a solve
  // stopped by maxiter before its state said done closes here)
  if (launched > 0 && speculative_close() && hs.all_done) return PF_OK;
  if (nm && launched > 0) {
    // x = x0 + M^-1 z: a one-stage stencil, on the single-halo tiled pass
    halo(pl, s, {{z, ncomp}});
    launch_tiled<kTrans, 4>(tg, tgrid, s, a, bv, 0, (int64_t)n, st, w, z,
                            nullptr, 0, 0, x);
  }
  launch(k_bi_finish, ge, kBlock, s, x, n, rg, st);
  halo(pl, s, {{x, ncomp}});
  if (tinit)
    launch_tiled<kTrans, 3>(tg, tgrid, s, a, bv, 0, (int64_t)n, st, w, x, b,
                            ncomp);
  else
  launch(k_true_res<V>, gr, kBlock, s, v, a, kTrans ? 1 : 0, ncomp, b, x, st,
                                      w.partials, w.counters);
  PF_LAUNCH_CHECK("bicgstab finish");
  return read_state(pl, st, &hs, s);
}

}  // namespace

extern "C" int pf_bicgstab_solve(const pf_plan *plan, const double *a,
                                 int32_t transpose, int32_t ncomp,
                                 const double *b, double *x, int32_t has_x0,
                                 double tol, int32_t maxiter, int32_t precond,
                                 void *workspace,
                                 pf_solver_report *reports_host,
                                 void *stream) {
  if (!plan || !a || !b || !x || !workspace || !reports_host || ncomp < 1 ||
      ncomp > 3 || maxiter < 0) {
    set_error("pf_bicgstab_solve: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  if (ncomp > pl.d.dim) {
    set_error("pf_bicgstab_solve: ncomp exceeds the workspace sizing");
    return PF_ERR_ARG;
  }
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  SolverState *st = reinterpret_cast<SolverState *>(w.solver);
  cudaStream_t s = S(stream);
  const int32_t n = (int32_t)pl.d.n;
  return dispatch(pl, [&](auto v) {
    using V = decltype(v);
    auto core = [&](SolverState &hs, double tl, int mi, int pc, unsigned mask,
                    int fresh) {
      return transpose
                 ? bi_core<V, true>(pl, v, w, st, hs, a, b, x, ncomp, tl, mi,
                                    pc, mask, fresh, s)
                 : bi_core<V, false>(pl, v, w, st, hs, a, b, x, ncomp, tl, mi,
                                     pc, mask, fresh, s);
    };
    if (!has_x0)
      PF_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n * ncomp, s));
    SolverState hs;
    int rc = core(hs, tol, maxiter, precond, 0x7u, 1);
    if (rc) return rc;
    pf_solver_report rep[3];
    double bnorm[3];
    unsigned redo = 0;
    for (int q = 0; q < ncomp; ++q) {
      const CompState &c = hs.c[q];
      bnorm[q] = c.bnorm;
      rep[q].fallback_used = 0;
      rep[q].breakdown = c.fail;
      if (c.zero_rhs) {
        rep[q].converged = 1;
        rep[q].iterations = 0;
        rep[q].residual = 0.0;
        continue;
      }
      const bool ok = c.converged && c.true_res <= 10.0 * c.tol_abs;
      rep[q].converged = ok;
      rep[q].iterations = c.iter;
      rep[q].residual = (c.converged ? c.true_res : c.res) / c.bnorm;
      if (!ok && precond) redo |= 1u << q;
    }
    if (redo) {
      for (int q = 0; q < ncomp; ++q)
        if ((redo >> q) & 1u)
          PF_CUDA(cudaMemsetAsync(x + (int64_t)q * n, 0, sizeof(double) * n, s));
      rc = core(hs, tol, 2 * maxiter, 0, redo, 0);
      if (rc) return rc;
      for (int q = 0; q < ncomp; ++q) {
        if (!((redo >> q) & 1u)) continue;
        const CompState &c = hs.c[q];
        rep[q].fallback_used = 1;
        rep[q].breakdown = c.fail;
        rep[q].iterations += c.iter;
        rep[q].converged = c.converged && c.true_res <= 10.0 * c.tol_abs;
        rep[q].residual = (c.converged ? c.true_res : c.res) / bnorm[q];
      }
    }
    for (int q = 0; q < ncomp; ++q) reports_host[q] = rep[q];
    return PF_OK;
  });
}

// ---------------------------------------------------------------------------
// live per-kernel timing of the CG iteration on a real operator (bench.py
// roofline): runs `iters` iterations that never converge (tol = 0) and
// times each of the three iteration kernels with CUDA events on `stream`.

extern "C" int pf_cg_profile(const pf_plan *plan, const double *a,
                             const double *b, int32_t iters, int32_t precond,
                             void *workspace, void *mg_workspace,
                             double *ms_host, void *stream) {
  if (!plan || !a || !b || !workspace || !ms_host || iters < 1 ||
      precond < 0 || precond > 2) {
    set_error("pf_cg_profile: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  MgHierarchy mg;
  if (precond == 2) {
    if (!pl.has_mg || !mg_workspace) {
      set_error("pf_cg_profile: multigrid unavailable");
      return PF_ERR_UNSUPPORTED;
    }
    mg = pl.mg;
    mg_bind(mg, mg_workspace);
  }
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  SolverState *st = reinterpret_cast<SolverState *>(w.solver);
  cudaStream_t s = S(stream);
  const int32_t n = (int32_t)pl.d.n;
  double *r = w.vecs, *p = w.vecs + n, *q = w.vecs + 2 * (int64_t)n;
  double *bp = w.vecs + 3 * (int64_t)n, *z = w.vecs + 4 * (int64_t)n;
  double *x = w.vecs + 5 * (int64_t)n;
  const int *done = &st->all_done;
  return dispatch(pl, [&](auto v) {
    using V = decltype(v);
    const int ge = grid_for(pl.i1 - pl.i0), gr = std::min(ge, pl.red_blocks);
  const Rng rg = plan_range(pl);
    PF_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    // room for the timed iterations plus the graph-replay measurement
    launch(k_cg_reset, 1, 1, s, st, 2 * iters + 2 * kGraphIters + 1, precond,
           1, 0.0, 1);
    launch(k_cg_bsum, gr, kBlock, s, b, 1.0, rg, st, w.partials, w.counters);
    launch(k_cg_bproj, gr, kBlock, s, b, 1.0, bp, rg, st, w.partials,
           w.counters);
    launch(k_cg_resid<V>, gr, kBlock, s, v, a, bp, x, r, st, w.partials,
           w.counters);
    launch(k_cg_rproj, gr, kBlock, s, a, r, rg, st, w.partials, w.counters);
    if (precond == 2) {
      const CgFuse fuse{st, w.partials, w.counters, 1};
      int rc = mg_apply(mg, r, z, s, done, nullptr, &fuse, pl.red_blocks, &pl);
      if (rc) return rc;
    }
    // the tiled fused direction update + SpMV where production runs it
    TileGeo tgc;
    const bool cgt = precond == 2 && cg_tiled(pl, &mg, tgc);
    double *p1 = w.vecs + 6 * (int64_t)n;
    if (!cgt)
      launch(k_cg_pinit, ge, kBlock, s, a, r, (const double *)z, p, rg, st);
    // events: 0 start | 1 spmv | 2 update | 3..8 mg level-0 marks | 9 zsum |
    // 10 pupdate (tiled: folded into the spmv)
    cudaEvent_t ev[11];
    for (auto &e : ev) PF_CUDA(cudaEventCreate(&e));
    double tot[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < iters; ++k) {
      if (!cgt) halo(pl, s, {{p, 1}});
      PF_CUDA(cudaEventRecord(ev[0], s));
      if (cgt)
        launch_cg_spmv_pt(tgc, pl, mg.lv[0], z, p, p1, q, st, w, s);
      else if (precond == 2)
        launch(k_cg_spmv_faces, gr, kBlock, s, mg.lv[0], rg, (const double *)p,
               q, st, w.partials, w.counters);
      else
        launch(k_cg_spmv<V>, gr, kBlock, s, v, a, p, q, st, w.partials,
               w.counters);
      PF_CUDA(cudaEventRecord(ev[1], s));
      if (cgt)
        launch(k_cg_update_pt, gr, kBlock, s, (const double *)p,
               (const double *)p1, (const double *)q, x, r, rg, st,
               w.partials, w.counters);
      else
        launch(k_cg_update, gr, kBlock, s, a, p, q, x, r, rg, st, w.partials,
               w.counters);
      PF_CUDA(cudaEventRecord(ev[2], s));
      if (precond == 2) {
        // as in production: the z-sums ride in the last smoothing pass, so
        // the zsum slot measures ~0
        const CgFuse fuse{st, w.partials, w.counters, 0};
        int rc = mg_apply(mg, r, z, s, done, ev + 3, &fuse, pl.red_blocks, &pl);
        if (rc) return rc;
      } else {
        for (int j = 3; j < 9; ++j) PF_CUDA(cudaEventRecord(ev[j], s));
      }
      PF_CUDA(cudaEventRecord(ev[9], s));
      if (!cgt)
        launch(k_cg_pupdate, ge, kBlock, s, a, r, (const double *)z, p, rg, st);
      PF_CUDA(cudaEventRecord(ev[10], s));
      PF_CUDA(cudaEventSynchronize(ev[10]));
      // spmv, update, [mg: smooth0, restrict, coarse, prolong, smooth2],
      // zsum, pupdate, whole iteration
      const int from[9] = {0, 1, 3, 4, 5, 6, 7, 8, 9};
      const int to[9] = {1, 2, 4, 5, 6, 7, 8, 9, 10};
      for (int j = 0; j < 9; ++j) {
        float ms = 0.f;
        PF_CUDA(cudaEventElapsedTime(&ms, ev[from[j]], ev[to[j]]));
        tot[j] += ms;
      }
      float ms = 0.f;
      PF_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[10]));
      tot[9] += ms;
    }
    // [10]: the production path -- iterations replayed from the cached
    // CUDA graph (multigrid only)
    double graph_ms = 0.0;
    if (precond == 2) {
      cudaGraphExec_t exec;
      unsigned long long nk = 0;
      int rc = mg_graph(pl, w, st, &mg, x, &exec, &nk);
      if (rc) return rc;
      const int reps = std::max(1, iters / kGraphIters);
      PF_CUDA(cudaEventRecord(ev[0], s));
      for (int k = 0; k < reps; ++k) {
        PF_CUDA(cudaGraphLaunch(exec, s));
        g_launches.fetch_add(nk, std::memory_order_relaxed);
      }
      PF_CUDA(cudaEventRecord(ev[1], s));
      PF_CUDA(cudaEventSynchronize(ev[1]));
      float ms = 0.f;
      PF_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      graph_ms = ms / (reps * kGraphIters);
    }
    for (auto &e : ev) cudaEventDestroy(e);
    SolverState hs;
    int rc = read_state(pl, st, &hs, s);
    if (!rc) rc = comm_check(pl, s);
    if (rc) return rc;
    if (hs.all_done) {
      set_error("pf_cg_profile: iteration stopped early (breakdown)");
      return PF_ERR_ARG;
    }
    for (int j = 0; j < 10; ++j) ms_host[j] = tot[j] / iters;
    ms_host[10] = graph_ms;
    ms_host[11] = cgt ? 1.0 : 0.0;
    return PF_OK;
  });
}

// ---------------------------------------------------------------------------
// live per-pass timing of the batched BiCGStab iteration (bench.py roofline)

extern "C" int pf_bicgstab_profile(const pf_plan *plan, const double *a,
                                   int32_t transpose, int32_t ncomp,
                                   const double *b, int32_t iters,
                                   void *workspace, double *ms_host,
                                   void *stream) {
  if (!plan || !a || !b || !workspace || !ms_host || iters < 1 || ncomp < 1 ||
      ncomp > 3) {
    set_error("pf_bicgstab_profile: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  if (ncomp > pl.d.dim) {
    set_error("pf_bicgstab_profile: ncomp exceeds the workspace sizing");
    return PF_ERR_ARG;
  }
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  SolverState *st = reinterpret_cast<SolverState *>(w.solver);
  cudaStream_t s = S(stream);
  const int32_t n = (int32_t)pl.d.n;
  const int64_t len = (int64_t)ncomp * n;
  // x lives past the seven solver vectors, 1 / diag and z
  double *x = w.vecs + 9 * len;
  double *z = w.vecs + 8 * len;
  return dispatch(pl, [&](auto v) {
    using V = decltype(v);
    BiVecs bv;
    bv.r = w.vecs;
    bv.rhat = w.vecs + len;
    bv.t = w.vecs + 2 * len;
    bv.p[0] = w.vecs + 3 * len;
    bv.p[1] = w.vecs + 4 * len;
    bv.v[0] = w.vecs + 5 * len;
    bv.v[1] = w.vecs + 6 * len;
    bv.dinv = w.vecs + 7 * len;
    const int gr = std::min(grid_for(pl.i1 - pl.i0), pl.red_blocks);
    const Rng rg = plan_range(pl);
    TileGeo tg, tgn;
    const bool tiled = tile_geo(pl, v, tg);
    const int tgrid = tiled ? std::min(tg.ntiles, pl.red_blocks) : 0;
    // the production preconditioner, as linalg.py picks it: Neumann-2 where
    // its tiled passes run (slab plans of several ranks: only when
    // PF_MOMENTUM_PRECOND=neumann2), Jacobi when PF_MOMENTUM_PRECOND=jacobi
    TileGeo tge;
    const char *mp = getenv("PF_MOMENTUM_PRECOND");
    const bool multi = pl.slab && pl.d.slab_world > 1;
    const bool nm = (mp ? std::string(mp) == "neumann2" : !multi) &&
                    nm_geo(pl, v, tgn, &tge);
    const int ngrid = nm ? std::min(tgn.ntiles, nm_minb() * pl.num_sms) : 0;
    const int egrid = nm ? std::min(tge.ntiles, nm_minb() * pl.num_sms) : 0;
    double *qg = pl.slab ? w.vecs + 10 * len : nullptr;
    PF_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * len, s));
    // tol 0: the recurrence never converges inside the timed iterations
    launch(k_bi_reset, 1, 1, s, st, ncomp, iters + 1, nm ? kPrecondNeumann2 : 1,
           0.0, 1, 0x7u);
    launch(k_bi_bnorm, gr, kBlock, s, b, n, rg, st, w.partials, w.counters);
    halo(pl, s, {{x, ncomp}});
    if (transpose)
      launch(k_bi_init<V, true>, gr, kBlock, s, v, a, b, (const double *)x,
             bv, st, w.partials, w.counters);
    else
      launch(k_bi_init<V, false>, gr, kBlock, s, v, a, b, (const double *)x,
             bv, st, w.partials, w.counters);
    halo(pl, s, {{bv.v[0], ncomp}, {bv.dinv, 1}});
    cudaEvent_t ev[4];
    for (auto &e : ev) PF_CUDA(cudaEventCreate(&e));
    double tot[4] = {0, 0, 0, 0};
    if (nm) {
      // Neumann-2: iteration 0 (pv) untimed, then per iteration the merged
      // x/r + pv pass and the st pass (no separate x/r pass)
      bv.rb[0] = bv.r;
      bv.rb[1] = w.vecs + 11 * len;
      bv.z = z;
      auto one = [&](int k, bool timed) -> int {
        const int par = k & 1;
        if (timed) PF_CUDA(cudaEventRecord(ev[0], s));
        if (k == 0) {
          halo(pl, s, {{bv.rb[0], ncomp}, {bv.p[par], ncomp}});
          if (qg) {
            if (transpose)
              launch_nm<true, 0>(tge, egrid, s, a, bv, par, (int64_t)n, st, w,
                                 1, nullptr, nullptr, nullptr, qg);
            else
              launch_nm<false, 0>(tge, egrid, s, a, bv, par, (int64_t)n, st,
                                  w, 1, nullptr, nullptr, nullptr, qg);
            halo(pl, s, {{qg, ncomp}});
          }
          if (transpose)
            launch_nm<true, 0>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w, 1,
                               nullptr, nullptr, qg);
          else
            launch_nm<false, 0>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w,
                                1, nullptr, nullptr, qg);
        } else {
          const int rp = (k - 1) & 1;
          halo(pl, s, {{bv.rb[rp], ncomp}, {bv.p[par], ncomp}, {bv.t, ncomp}});
          if (qg) {
            if (transpose)
              launch_nm<true, 3>(tge, egrid, s, a, bv, par, (int64_t)n, st, w,
                                 0, nullptr, nullptr, nullptr, qg, rp);
            else
              launch_nm<false, 3>(tge, egrid, s, a, bv, par, (int64_t)n, st,
                                  w, 0, nullptr, nullptr, nullptr, qg, rp);
            halo(pl, s, {{qg, ncomp}});
          }
          if (transpose)
            launch_nm<true, 3>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w, 0,
                               nullptr, nullptr, qg, nullptr, rp);
          else
            launch_nm<false, 3>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w,
                                0, nullptr, nullptr, qg, nullptr, rp);
        }
        if (timed) PF_CUDA(cudaEventRecord(ev[1], s));
        halo(pl, s, {{bv.v[par ^ 1], ncomp}, {bv.rb[par], ncomp}});
        if (qg) {
          if (transpose)
            launch_nm<true, 1>(tge, egrid, s, a, bv, par, (int64_t)n, st, w, 0,
                               nullptr, nullptr, nullptr, qg, par);
          else
            launch_nm<false, 1>(tge, egrid, s, a, bv, par, (int64_t)n, st, w,
                                0, nullptr, nullptr, nullptr, qg, par);
          halo(pl, s, {{qg, ncomp}});
        }
        if (transpose)
          launch_nm<true, 1>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w, 0,
                             nullptr, nullptr, qg, nullptr, par);
        else
          launch_nm<false, 1>(tgn, ngrid, s, a, bv, par, (int64_t)n, st, w, 0,
                              nullptr, nullptr, qg, nullptr, par);
        if (!timed) return PF_OK;
        PF_CUDA(cudaEventRecord(ev[2], s));
        PF_CUDA(cudaEventRecord(ev[3], s));
        PF_CUDA(cudaEventSynchronize(ev[3]));
        for (int j = 0; j < 3; ++j) {
          float ms = 0.f;
          PF_CUDA(cudaEventElapsedTime(&ms, ev[j], ev[j + 1]));
          tot[j] += ms;
        }
        float ms = 0.f;
        PF_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[3]));
        tot[3] += ms;
        return PF_OK;
      };
      int rc = one(0, false);
      for (int k = 1; k <= iters && !rc; ++k) rc = one(k, true);
      if (rc) return rc;
    }
    for (int k = 0; k < iters && !nm; ++k) {
      const int par = k & 1;
      halo(pl, s, {{bv.r, ncomp}, {bv.p[par], ncomp}});
      PF_CUDA(cudaEventRecord(ev[0], s));
      if (tiled && transpose)
        launch_tiled<true, 0>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w);
      else if (tiled)
        launch_tiled<false, 0>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w);
      else if (transpose)
        launch(k_bi_pv<V, true>, gr, kBlock, s, v, a, bv, par, st, w.partials,
               w.counters);
      else
        launch(k_bi_pv<V, false>, gr, kBlock, s, v, a, bv, par, st,
               w.partials, w.counters);
      halo(pl, s, {{bv.v[par ^ 1], ncomp}});
      PF_CUDA(cudaEventRecord(ev[1], s));
      if (tiled && transpose)
        launch_tiled<true, 1>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w);
      else if (tiled)
        launch_tiled<false, 1>(tg, tgrid, s, a, bv, par, (int64_t)n, st, w);
      else if (transpose)
        launch(k_bi_st<V, true>, gr, kBlock, s, v, a, bv, par, st, w.partials,
               w.counters);
      else
        launch(k_bi_st<V, false>, gr, kBlock, s, v, a, bv, par, st,
               w.partials, w.counters);
      PF_CUDA(cudaEventRecord(ev[2], s));
      launch(k_bi_xr<false>, gr, kBlock, s, a, bv, par, x, n, rg, st,
               w.partials, w.counters, 0);
      PF_CUDA(cudaEventRecord(ev[3], s));
      PF_CUDA(cudaEventSynchronize(ev[3]));
      for (int j = 0; j < 3; ++j) {
        float ms = 0.f;
        PF_CUDA(cudaEventElapsedTime(&ms, ev[j], ev[j + 1]));
        tot[j] += ms;
      }
      float ms = 0.f;
      PF_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[3]));
      tot[3] += ms;
    }
    for (auto &e : ev) cudaEventDestroy(e);
    SolverState hs;
    int rc = read_state(pl, st, &hs, s);
    if (!rc) rc = comm_check(pl, s);
    if (rc) return rc;
    if (hs.all_done) {
      set_error("pf_bicgstab_profile: iteration stopped early (breakdown)");
      return PF_ERR_ARG;
    }
    for (int j = 0; j < 4; ++j) ms_host[j] = tot[j] / iters;
    ms_host[4] = nm ? kPrecondNeumann2 : 1;
    return PF_OK;
  });
}
