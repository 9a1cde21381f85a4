// cross.cu -- lagged non-orthogonal fluxes and their adjoints.
//
// On grids whose metric tensor alpha has off-diagonal entries, the PISO
// step moves the cross-derivative fluxes to the right-hand sides and lags
// them (S/piso.py:322-353 momentum, 375-392 tangential boundary flux,
// 431-449 pressure); extra outer iterations (StepConfig.nonortho_correctors)
// refresh them.  The adjoints are S/adjoint.py:156-233.  Every transpose is
// a gather over the back face, as in adjoint.cu.
#include <algorithm>

#include "common.cuh"

namespace pf {

// one-sided wide gradient of component c of field f at cell i along every
// axis (wide_grad "onesided", S/piso.py:172-209): weight 1/2 with both
// neighbours, else a full one-sided difference with the cell itself
template <class V>
__device__ __forceinline__ void onesided_grad(const V &v,
                                              const Face (&fc)[2 * V::kDim],
                                              const double *__restrict__ f,
                                              int32_t i,
                                              double (&g)[V::kDim]) {
#pragma unroll
  for (int a = 0; a < V::kDim; ++a) {
    const Face &lo = fc[2 * a], &hi = fc[2 * a + 1];
    const double fi = f[i];
    const double vhi = hi.nb >= 0 ? f[hi.nb] : fi;
    const double vlo = lo.nb >= 0 ? f[lo.nb] : fi;
    const double w = (hi.nb >= 0 && lo.nb >= 0) ? 0.5 : 1.0;
    g[a] = w * (vhi - vlo);
  }
}

template <class V>
__device__ __forceinline__ void faces_of(const V &v, int32_t i,
                                         Face (&fc)[2 * V::kDim]) {
  const auto cell = v.topo.cell(i);
#pragma unroll
  for (int f = 0; f < 2 * V::kDim; ++f) fc[f] = v.topo.face(cell, f);
}

// weight of the one-sided gradient of cell i along axis a
template <class V>
__device__ __forceinline__ double onesided_w(const V &v, int32_t i, int a) {
  const auto cell = v.topo.cell(i);
  const Face lo = v.topo.face(cell, 2 * a), hi = v.topo.face(cell, 2 * a + 1);
  return (hi.nb >= 0 && lo.nb >= 0) ? 0.5 : 1.0;
}

// ---------------------------------------------------------------------------
// forward: momentum cross flux  x[a][c] = nu sum_{k != a} alpha_ak g_kc

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_xmom_x(V v, const double *__restrict__ u, double nu,
             double *__restrict__ x) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, i, fc);
  double g[D][D];  // g[k][c]
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double gc[D];
    onesided_grad(v, fc, u + c * n, i, gc);
#pragma unroll
    for (int k = 0; k < D; ++k) g[k][c] = gc[k];
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double full = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) full += v.AF(a, k, i) * g[k][c];
      x[(int64_t)(a * D + c) * n + i] = nu * full - nu * v.AF(a, a, i) * g[a][c];
    }
  }
}

// rhs[c] += (sum_faces N (x[i,a,c] + sign x[nb, perm a, c]) / 2) / J
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_xmom_div(V v, const double *__restrict__ x, double *__restrict__ rhs) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, i, fc);
  double out[D];
#pragma unroll
  for (int c = 0; c < D; ++c) out[c] = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    if (fc[f].nb < 0) continue;
    const int a = f >> 1;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double xn = x[(int64_t)(fc[f].ax * D + c) * n + fc[f].nb];
      out[c] += nsgn * (0.5 * (x[(int64_t)(a * D + c) * n + i] +
                               (fc[f].neg ? -xn : xn)));
    }
  }
  const double J = v.J(i);
#pragma unroll
  for (int c = 0; c < D; ++c) rhs[c * n + i] += out[c] / J;
}

// ---------------------------------------------------------------------------
// forward: pressure cross flux  x[a] = A^-1 sum_{k != a} alpha_ak g_k(p)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_xp_x(V v, const double *__restrict__ c, const double *__restrict__ p,
           double *__restrict__ x) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, i, fc);
  double g[D];
  onesided_grad(v, fc, p, i, g);
  const double ainv = 1.0 / c[i];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double full = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) full += v.AF(a, k, i) * g[k];
    x[(int64_t)a * n + i] = ainv * full - ainv * v.AF(a, a, i) * g[a];
  }
}

// b = b0 - sum_faces N (x[i,a] + sign x[nb, perm a]) / 2
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_xp_div(V v, const double *__restrict__ x, const double *__restrict__ b0,
             double *__restrict__ b) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, i, fc);
  double out = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    if (fc[f].nb < 0) continue;
    const int a = f >> 1;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    const double xn = x[(int64_t)fc[f].ax * n + fc[f].nb];
    out += nsgn * (0.5 * (x[(int64_t)a * n + i] + (fc[f].neg ? -xn : xn)));
  }
  b[i] = b0[i] - out;
}

// ---------------------------------------------------------------------------
// adjoint helpers: the face-mean gather (fetch_axis_trailing_adjoint) and
// the one-sided wide-gradient adjoint (wide_grad_adjoint "onesided")

// cot_x[a] at cell j from cell values cv (scaled by scale_of(cell)), over own
// faces and the neighbours' back faces (S/adjoint.py:166-173, 194-200)
template <class V, class Val>
__device__ __forceinline__ void face_mean_gather(const V &v, int32_t j,
                                                 const Face (&fc)[2 * V::kDim],
                                                 Val val,
                                                 double (&cx)[V::kDim]) {
#pragma unroll
  for (int a = 0; a < V::kDim; ++a) cx[a] = 0.0;
  const double cj = val(j);
#pragma unroll
  for (int f = 0; f < 2 * V::kDim; ++f) {
    if (fc[f].nb < 0) continue;
    const int a = f >> 1;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    cx[a] += 0.5 * nsgn * cj;
    const int fb = back_face(fc[f], f & 1);
    const double nsb = (fb & 1) ? 1.0 : -1.0;
    const double cf = 0.5 * nsb * val(fc[f].nb);
    cx[a] += fc[f].neg ? -cf : cf;
  }
}

// dphi[j] = sum over the one-sided wide-gradient stencils touching j of the
// cotangent cg[cell][axis] (component stride D*n when cg holds components)
template <class V>
__device__ __forceinline__ double onesided_adj_gather(
    const V &v, int32_t j, const Face (&fc)[2 * V::kDim],
    const double *__restrict__ cg, int64_t ax_stride) {
  constexpr int D = V::kDim;
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const bool hi = fc[2 * a + 1].nb >= 0, lo = fc[2 * a].nb >= 0;
    const double w = (hi && lo) ? 0.5 : 1.0;
    const double c = w * cg[(int64_t)a * ax_stride + j];
    if (!hi) acc += c;   // ghost of a missing neighbour lands on the cell
    if (!lo) acc -= c;
  }
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    if (fc[f].nb < 0) continue;
    const int32_t i = fc[f].nb;
    const int fb = back_face(fc[f], f & 1);
    const int ab = fb >> 1;
    const double c = onesided_w(v, i, ab) * cg[(int64_t)ab * ax_stride + i];
    acc += (fb & 1) ? c : -c;
  }
  return acc;
}

// ---------------------------------------------------------------------------
// adjoint of the pressure cross flux (_adj_pressure_cross, S/adjoint.py:
// 156-178): stage 1 per cell -> dA, cot_g;  stage 2 gather -> dp_prev

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_axp_cell(V v, const double *__restrict__ c, const double *__restrict__ p,
               const double *__restrict__ cot_out, double cs,
               double *__restrict__ da, double *__restrict__ cot_g) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, j, fc);
  double cx[D];
  face_mean_gather(v, j, fc, [&](int32_t k) { return cs * cot_out[k]; }, cx);
  double g[D];
  onesided_grad(v, fc, p, j, g);
  double dain = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double full = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) full += v.AF(a, k, j) * g[k];
    dain += cx[a] * (full - v.AF(a, a, j) * g[a]);
  }
  const double ainv = 1.0 / c[j];
  da[j] += -(ainv * ainv) * dain;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) s += v.AF(a, k, j) * (ainv * cx[a]);
    cot_g[(int64_t)k * n + j] = s - v.AF(k, k, j) * (ainv * cx[k]);
  }
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_adj_onesided(V v, const double *__restrict__ cot_g, int ncomp,
                   double *__restrict__ out, int accumulate) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  Face fc[2 * D];
  faces_of(v, j, fc);
  for (int q = 0; q < ncomp; ++q) {
    // component q of an (axis, component) field lives at (a*ncomp + q)*n
    const double r = onesided_adj_gather(v, j, fc, cot_g + (int64_t)q * n,
                                         (int64_t)ncomp * n);
    if (accumulate)
      out[(int64_t)q * n + j] += r;
    else
      out[(int64_t)q * n + j] = r;
  }
}

// ---------------------------------------------------------------------------
// adjoint of the momentum cross flux (_adj_momentum_cross, S/adjoint.py:
// 181-205): per cell cot_x, nu sensitivity, cot_g

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_axmom_cell(V v, const double *__restrict__ u, double nu,
                 const double *__restrict__ cot_out,
                 double *__restrict__ cot_g, double *dnu, double *partials,
                 unsigned *counter) {
  constexpr int D = V::kDim;
  const int64_t n = v.n;
  double acc[1] = {0.0};
  RANGE_LOOP(j, v.rng()) {
    Face fc[2 * D];
    faces_of(v, j, fc);
    double cx[D][D];  // cx[a][c]
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double col[D];
      face_mean_gather(
          v, j, fc,
          [&](int32_t k) { return cot_out[(int64_t)c * n + k] / v.J(k); },
          col);
#pragma unroll
      for (int a = 0; a < D; ++a) cx[a][c] = col[a];
    }
    double g[D][D];  // g[k][c]
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double gc[D];
      onesided_grad(v, fc, u + c * n, j, gc);
#pragma unroll
      for (int k = 0; k < D; ++k) g[k][c] = gc[k];
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double full = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) full += v.AF(a, k, j) * g[k][c];
        acc[0] += cx[a][c] * (nu * full - nu * v.AF(a, a, j) * g[a][c]);
      }
#pragma unroll
    for (int k = 0; k < D; ++k)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) s += v.AF(a, k, j) * cx[a][c];
        cot_g[(int64_t)(k * D + c) * n + j] =
            nu * s - nu * v.AF(k, k, j) * cx[k][c];
      }
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) *dnu += tot[0] / nu;
}

}  // namespace pf

// ===========================================================================
// C ABI

using namespace pf;

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }
static const Plan &P(const pf_plan *p) {
  return *reinterpret_cast<const Plan *>(p);
}

#define PF_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) {            \
      ::pf::set_error(msg);   \
      return PF_ERR_ARG;      \
    }                         \
  } while (0)

#define PF_REQUIRE_CROSS(pl)                                             \
  PF_REQUIRE((pl).d.alpha_full, "non-orthogonal terms need a plan built " \
                                "with the full metric tensor")

extern "C" int pf_momentum_cross_rhs(const pf_plan *plan, const double *u,
                                     double nu, double *rhs_inout,
                                     void *workspace, void *stream) {
  PF_REQUIRE(plan && u && rhs_inout && workspace,
             "pf_momentum_cross_rhs: null argument");
  const Plan &pl = P(plan);
  PF_REQUIRE_CROSS(pl);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    double *x = w.vecs;  // (d*d, n)
    launch(k_xmom_x<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, u, nu,
           x);
    launch(k_xmom_div<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v,
           (const double *)x, rhs_inout);
    PF_LAUNCH_CHECK("momentum_cross_rhs");
    return PF_OK;
  });
}

extern "C" int pf_pressure_cross_rhs(const pf_plan *plan, const double *c,
                                     const double *p_prev, const double *b0,
                                     double *b_out, void *workspace,
                                     void *stream) {
  PF_REQUIRE(plan && c && p_prev && b0 && b_out && workspace,
             "pf_pressure_cross_rhs: null argument");
  const Plan &pl = P(plan);
  PF_REQUIRE_CROSS(pl);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    double *x = w.vecs;  // (d, n)
    launch(k_xp_x<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c,
           p_prev, x);
    launch(k_xp_div<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v,
           (const double *)x, b0, b_out);
    PF_LAUNCH_CHECK("pressure_cross_rhs");
    return PF_OK;
  });
}

extern "C" int pf_adj_pressure_cross(const pf_plan *plan, const double *c,
                                     const double *p_prev,
                                     const double *cot_out, double cot_scale,
                                     double *da, double *dp_prev,
                                     void *workspace, void *stream) {
  PF_REQUIRE(plan && c && p_prev && cot_out && da && dp_prev && workspace,
             "pf_adj_pressure_cross: null argument");
  const Plan &pl = P(plan);
  PF_REQUIRE_CROSS(pl);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    double *cot_g = w.vecs;  // (d, n)
    launch(k_axp_cell<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c,
           p_prev, cot_out, cot_scale, da, cot_g);
    launch(k_adj_onesided<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v,
           (const double *)cot_g, 1, dp_prev, 0);
    PF_LAUNCH_CHECK("adj_pressure_cross");
    return PF_OK;
  });
}

extern "C" int pf_adj_momentum_cross(const pf_plan *plan, const double *u,
                                     double nu, const double *cot_out,
                                     double *du_cross, int32_t accumulate,
                                     double *dnu_dev, void *workspace,
                                     void *stream) {
  PF_REQUIRE(plan && u && cot_out && du_cross && dnu_dev && workspace,
             "pf_adj_momentum_cross: null argument");
  const Plan &pl = P(plan);
  PF_REQUIRE_CROSS(pl);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    constexpr int D = decltype(v)::kDim;
    double *cot_g = w.vecs;  // (d*d, n) at [(k*D + c) * n]
    const int g = std::min(grid_for(v.owned()), pl.red_blocks);
    launch(k_axmom_cell<decltype(v)>, g, kBlock, S(stream), v, u, nu, cot_out,
           cot_g, dnu_dev, w.partials, w.counters);
    launch(k_adj_onesided<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v,
           (const double *)cot_g, D, du_cross, (int)accumulate);
    PF_LAUNCH_CHECK("adj_momentum_cross");
    return PF_OK;
  });
}

__global__ void __launch_bounds__(kBlock)
    k_axpy(double alpha, const double *__restrict__ x, double *__restrict__ y,
           int64_t len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) y[i] += alpha * x[i];
}

extern "C" int pf_axpy(const pf_plan *plan, double alpha, const double *x,
                       double *y, int64_t len, void *stream) {
  PF_REQUIRE(plan && x && y && len >= 0, "pf_axpy: bad argument");
  if (len == 0) return PF_OK;
  launch(k_axpy, grid_for(len), kBlock, S(stream), alpha, x, y, len);
  PF_LAUNCH_CHECK("axpy");
  return PF_OK;
}
