// adjoint.cu -- discrete adjoint stage kernels (S/adjoint.py:78-340).
//
// The reference scatters neighbour contributions with np.add.at; here every
// transpose is evaluated as a GATHER: cell j visits each neighbour i across
// its face f' and pulls the contribution i made through its back face
// (the face of i that points at j, S/mesh.py:393-397).  Each output is
// written by exactly one thread in a fixed order, so the backward pass is
// bitwise reproducible (T/test_adjoint.py:394-406) without atomics.
#include "common.cuh"

namespace pf {

#define GRID_LOOP(i, n)                                                  \
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (n);       \
       i += gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// backward_correct_velocity (S/adjoint.py:78-91) -- stage 1: per cell
// cot_gp^a = T[a,:] . (-A^-1 cu) and dA += (cu . T^t g_mirror(p)) / A^2

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_cv_cell(V v, const double *__restrict__ p,
                  const double *__restrict__ c, const double *__restrict__ cu,
                  double *__restrict__ da, double *__restrict__ cot_gp, int ow) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  const double pi = p[i];
  double g[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const Face lo = v.topo.face(cell, 2 * a);
    const Face hi = v.topo.face(cell, 2 * a + 1);
    const double vhi = hi.nb >= 0 ? p[hi.nb] : pi;
    const double vlo = lo.nb >= 0 ? p[lo.nb] : pi;
    g[a] = 0.5 * (vhi - vlo);
  }
  const double ainv = 1.0 / c[i];
  double dot = 0.0;
  double cue[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double e = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) e += v.T(j, k, i) * g[j];
    const double cuk = cu[k * n + i];
    dot += cuk * e;
    cue[k] = -ainv * cuk;
  }
  if (ow)
    da[i] = dot * (ainv * ainv);
  else
    da[i] += dot * (ainv * ainv);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += v.T(a, k, i) * cue[k];
    cot_gp[a * n + i] = s;
  }
}

// stage 2: dp = wide_grad_adjoint(cot_gp, mirror) (S/piso.py:218-258)
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_cv_gather(V v, const double *__restrict__ cot_gp,
                    const double *__restrict__ extra, double *__restrict__ dp) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(j);
  double acc = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb >= 0) {
      const int fb = back_face(fc, f & 1);
      const double ci = cot_gp[(int64_t)(fb >> 1) * n + fc.nb];
      acc += (fb & 1) ? 0.5 * ci : -0.5 * ci;
    } else {
      // mirror ghost: the missing neighbour's weight lands on the cell
      const double cj = cot_gp[(int64_t)(f >> 1) * n + j];
      acc += (f & 1) ? 0.5 * cj : -0.5 * cj;
    }
  }
  if (extra) acc += extra[j];
  dp[j] = acc;
}

// ---------------------------------------------------------------------------
// pressure-matrix cotangent per face: dkf[f][i] += y_i (p_nb - p_i)
// (outer_on_pattern S/linalg.py:111-117 with the diagonal folded in the way
// backward_pressure_matrix S/adjoint.py:120-128 consumes it)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_p_outer(V v, const double *__restrict__ y,
                  const double *__restrict__ p, double *__restrict__ dkf,
                  int ow) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  const double yi = y[i], pi = p[i];
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (ow)
      dkf[(int64_t)f * n + i] = fc.nb >= 0 ? yi * p[fc.nb] - yi * pi : 0.0;
    else if (fc.nb >= 0)
      dkf[(int64_t)f * n + i] += yi * p[fc.nb] - yi * pi;
  }
}

// backward_pressure_matrix (S/adjoint.py:116-134): dA += -A^-2 g_ainv
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_p_matrix(V v, const double *__restrict__ c,
                   const double *__restrict__ dkf, double *__restrict__ da) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(j);
  double g = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) continue;
    const double aj = v.A(f >> 1, j);
    g += 0.5 * dkf[(int64_t)f * n + j] * aj;
    const int fb = back_face(fc, f & 1);
    g += 0.5 * dkf[(int64_t)fb * n + fc.nb] * aj;
  }
  const double ainv = 1.0 / c[j];
  da[j] += -(ainv * ainv) * g;
}

// ---------------------------------------------------------------------------
// _adj_divergence_rhs (S/adjoint.py:137-153)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_adj_div(V v, const double *__restrict__ cot_b, double cs,
              double *__restrict__ g_h, double *__restrict__ dbc) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(j);
  const double cb = cs * cot_b[j];
  double gf[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gf[a] = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    const int a = f >> 1;
    if (fc.nb >= 0) {
      const double nsgn = (f & 1) ? 1.0 : -1.0;
      gf[a] += 0.5 * nsgn * cb;
      // neighbour i's scatter through its back face lands on my axis a
      const int fb = back_face(fc, f & 1);
      const double nsb = (fb & 1) ? 1.0 : -1.0;
      const double cf = 0.5 * nsb * (cs * cot_b[fc.nb]);
      gf[a] += fc.neg ? -cf : cf;
    } else {
      const int32_t e = fc.bidx;
      const double nsgn = (f & 1) ? 1.0 : -1.0;
      const double coef = nsgn * __ldg(v.bjac + e) * cb;
#pragma unroll
      for (int k = 0; k < D; ++k)
        dbc[(int64_t)k * v.m + e] += coef * __ldg(v.bt + (int64_t)k * v.m + e);
    }
  }
  const double J = v.J(j);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) s += v.T(a, k, j) * gf[a];
    g_h[k * n + j] += J * s;
  }
}

// ---------------------------------------------------------------------------
// h-stage adjoint (S/adjoint.py:477-487): stage 1 per cell

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_h_cell(V v, const double *__restrict__ c,
                 const double *__restrict__ g_h, const double *__restrict__ h,
                 const double *__restrict__ u_hin, double *__restrict__ da,
                 double *__restrict__ g_rhs, double *__restrict__ dc,
                 double *__restrict__ cot_hu, int ow) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  const double ainv = 1.0 / c[i];
  double dot = 0.0;
  double chu[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const double gq = g_h[q * n + i];
    dot += gq * h[q * n + i];
    const double gr = ainv * gq;
    if (ow)
      g_rhs[q * n + i] = gr;
    else
      g_rhs[q * n + i] += gr;
    chu[q] = -gr;
    cot_hu[q * n + i] = -gr;
  }
  da[i] += -ainv * dot;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) {
      if (ow) dc[(int64_t)(1 + f) * n + i] = 0.0;
      continue;
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) s += chu[q] * u_hin[q * n + fc.nb];
    if (ow)
      dc[(int64_t)(1 + f) * n + i] = s;
    else
      dc[(int64_t)(1 + f) * n + i] += s;
  }
}

// stage 2: cu = (C^t - A) cot_hu, the off-diagonal transpose as a gather
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_h_gather(V v, const double *__restrict__ c,
                   const double *__restrict__ cot_hu, double *__restrict__ cu) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(j);
  double acc[D];
#pragma unroll
  for (int q = 0; q < D; ++q) acc[q] = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) continue;
    const int fb = back_face(fc, f & 1);
    const double coef = c[(int64_t)(1 + fb) * n + fc.nb];
#pragma unroll
    for (int q = 0; q < D; ++q) acc[q] += coef * cot_hu[q * n + fc.nb];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) cu[q * n + j] = acc[q];
}

// dC += outer(-y, u_star) on the pattern (S/adjoint.py:380)
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_bwd_mom_outer(V v, const double *__restrict__ y,
                    const double *__restrict__ us, double *__restrict__ dc) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  double yi[D];
  double dd = 0.0;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    yi[q] = -y[q * n + i];
    dd += yi[q] * us[q * n + i];
  }
  dc[i] += dd;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) continue;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) s += yi[q] * us[q * n + fc.nb];
    dc[(int64_t)(1 + f) * n + i] += s;
  }
}

// ---------------------------------------------------------------------------
// _adj_momentum_rhs (S/adjoint.py:236-268), orthogonal faces

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_adj_rhs_cells(V v, const double *__restrict__ cot, double dt,
                    double *__restrict__ du_n, int ow) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (ow)
      du_n[q * n + i] = cot[q * n + i] / dt;
    else
      du_n[q * n + i] += cot[q * n + i] / dt;
  }
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_adj_rhs_faces(V v, const double *__restrict__ cot,
                    const double *__restrict__ bc, double nu,
                    double *__restrict__ dbc, double *dnu, double *partials,
                    unsigned *counter) {
  constexpr int D = V::kDim;
  const int64_t n = v.n, m = v.m;
  double acc[1] = {0.0};
  GRID_LOOP(e, v.m) {
    const int32_t i = __ldg(v.bcell + e);
    // slab plans: entries of ghost-plane cells belong to a neighbour rank
    if (i < v.i0 || i >= v.i1) continue;
    const int bf = __ldg(v.bface + e);
    const int f = bf & 15, kind = bf >> 4;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    const double invj = v.IJ(i);
    const double fj = __ldg(v.bjac + e);
    double cr[D], ub[D], tr[D];
    double tu = 0.0, crub = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      cr[k] = cot[k * n + i];
      ub[k] = bc[k * m + e];
      tr[k] = __ldg(v.bt + k * m + e);
      tu += tr[k] * ub[k];
      crub += cr[k] * ub[k];
    }
    const double uflux = fj * tu;
    double coef;
    if (kind == PF_BKIND_DIRICHLET) {
      const double fa = __ldg(v.balpha + e);
      coef = (2.0 * nu * fa - uflux * nsgn) * invj;
      acc[0] += crub * 2.0 * fa * invj;
    } else {
      coef = -uflux * nsgn * invj;
    }
    const double cot_uflux = -nsgn * invj * crub;
#pragma unroll
    for (int k = 0; k < D; ++k)
      dbc[k * m + e] += cr[k] * coef + (cot_uflux * fj) * tr[k];
    if (kind == PF_BKIND_DIRICHLET && v.finfo) {
      const FaceGeo g = face_geo(v, e);
      if (g.active) {
        // _adj_boundary_cross (S/adjoint.py:215-233)
        double term[D];
        bcross_term(v, g, e, bc, term);
        const double sc = nsgn * nu / v.J(i);
        double dot = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) dot += cr[c] * (term[c] * sc);
        acc[0] += dot / nu;
        // face_grad_adjoint of fa * cot_pre along each tangential axis
        auto val = [&](int32_t e2, int q, int c) {
          const int32_t i2 = __ldg(v.bcell + e2);
          const double fa = __ldg(v.balpha_row +
                                  (int64_t)tang_axis(g.axis, q) * m + e2);
          return fa * (cot[c * n + i2] * (nsgn * nu / v.J(i2)));
        };
        for (int q = 0; q < g.ndim; ++q) {
          const int L = g.dims[q], j = g.j[q], st = g.st[q];
          if (L < 2) continue;
#pragma unroll
          for (int c = 0; c < D; ++c) {
            double o = 0.0;
            if (j - 1 >= 0) o += (j - 1 == 0) ? val(e - st, q, c)
                                              : 0.5 * val(e - st, q, c);
            if (j + 1 <= L - 1) o -= (j + 1 == L - 1) ? val(e + st, q, c)
                                                      : 0.5 * val(e + st, q, c);
            if (j == 0) o -= val(e, q, c);
            if (j == L - 1) o += val(e, q, c);
            dbc[c * m + e] += o;
          }
        }
      }
    }
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) *dnu += tot[0];
}

// ---------------------------------------------------------------------------
// _adj_assemble_momentum (S/adjoint.py:307-340)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_adj_assemble(V v, const double *__restrict__ dc, double nu,
                   double *__restrict__ du_n, double *dnu, double *partials,
                   unsigned *counter) {
  constexpr int D = V::kDim;
  const int64_t n = v.n;
  double acc[1] = {0.0};
  RANGE_LOOP(j, v.rng()) {
    const auto cell = v.topo.cell(j);
    const double cdj = dc[j];
    const double invj = v.IJ(j);
    double gf[D];
#pragma unroll
    for (int a = 0; a < D; ++a) gf[a] = 0.0;
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      const Face fc = v.topo.face(cell, f);
      const int a = f >> 1;
      if (fc.nb >= 0) {
        const double cot_off = dc[(int64_t)(1 + f) * n + j];
        const double cot_adv = cot_off + cdj;
        const double cot_visc = cdj - cot_off;
        acc[0] += cot_visc * 0.5 * (v.A(a, j) + v.A(fc.ax, fc.nb)) * invj;
        const double nsgn = (f & 1) ? 1.0 : -1.0;
        gf[a] += 0.5 * (0.5 * nsgn * invj * cot_adv);
        // neighbour's scatter through its back face
        const int32_t i = fc.nb;
        const int fb = back_face(fc, f & 1);
        const double ci = dc[(int64_t)(1 + fb) * n + i] + dc[i];
        const double nsb = (fb & 1) ? 1.0 : -1.0;
        const double cfm = 0.5 * (0.5 * nsb * (v.IJ(i)) * ci);
        gf[a] += fc.neg ? -cfm : cfm;
      } else {
        const int32_t e = fc.bidx;
        if ((__ldg(v.bface + e) >> 4) == PF_BKIND_DIRICHLET)
          acc[0] += cdj * 2.0 * __ldg(v.balpha + e) * invj;
      }
    }
    const double J = v.J(j);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) s += v.T(a, k, j) * gf[a];
      du_n[k * n + j] += J * s;
    }
  }
  double tot[1];
  if (grid_reduce<1>(acc, partials, counter, tot)) *dnu += tot[0];
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

extern "C" int pf_bwd_correct_velocity(const pf_plan *plan, const double *p,
                                       const double *c, const double *cu,
                                       double *da, double *cot_p,
                                       const double *extra_cot_p,
                                       int32_t overwrite, void *workspace,
                                       void *stream) {
  PF_REQUIRE(plan && p && c && cu && da && cot_p && workspace,
             "pf_bwd_correct_velocity: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    double *cot_gp = w.vecs;
    const int D = decltype(v)::kDim;
    halo(pl, S(stream), {{const_cast<double *>(p), 1}});
    launch(k_bwd_cv_cell<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, p, c, cu, da,
                                                           cot_gp, (int)overwrite);
    halo(pl, S(stream), {{cot_gp, D}});
    launch(k_bwd_cv_gather<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, cot_gp,
                                                             extra_cot_p, cot_p);
    PF_LAUNCH_CHECK("bwd_correct_velocity");
    return PF_OK;
  });
}

extern "C" int pf_bwd_pressure_outer(const pf_plan *plan, const double *y,
                                     const double *p, double *dkf,
                                     int32_t overwrite, void *stream) {
  PF_REQUIRE(plan && y && p && dkf, "pf_bwd_pressure_outer: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(p), 1}});
    launch(k_bwd_p_outer<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, y, p, dkf,
           (int)overwrite);
    PF_LAUNCH_CHECK("bwd_pressure_outer");
    return PF_OK;
  });
}

extern "C" int pf_bwd_pressure_matrix(const pf_plan *plan, const double *c,
                                      const double *dkf, double *da,
                                      void *stream) {
  PF_REQUIRE(plan && c && dkf && da, "pf_bwd_pressure_matrix: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream),
         {{const_cast<double *>(dkf), 2 * decltype(v)::kDim}});
    launch(k_bwd_p_matrix<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c, dkf, da);
    PF_LAUNCH_CHECK("bwd_pressure_matrix");
    return PF_OK;
  });
}

extern "C" int pf_adj_divergence_rhs(const pf_plan *plan, const double *cot_b,
                                     double cot_scale, double *g_h,
                                     double *dbc, void *stream) {
  PF_REQUIRE(plan && cot_b && g_h, "pf_adj_divergence_rhs: null argument");
  PF_REQUIRE(dbc || P(plan).d.m == 0, "pf_adj_divergence_rhs: null dbc");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(cot_b), 1}});
    launch(k_adj_div<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, cot_b, cot_scale,
                                                       g_h, dbc);
    PF_LAUNCH_CHECK("adj_divergence_rhs");
    return PF_OK;
  });
}

extern "C" int pf_bwd_h_stage(const pf_plan *plan, const double *c,
                              const double *g_h, const double *h,
                              const double *u_hin, double *da, double *g_rhs,
                              double *dc, double *cu_out, int32_t overwrite,
                              void *workspace, void *stream) {
  PF_REQUIRE(plan && c && g_h && h && u_hin && da && g_rhs && dc && cu_out &&
                 workspace,
             "pf_bwd_h_stage: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    double *cot_hu = w.vecs;
    const int D = decltype(v)::kDim;
    halo(pl, S(stream), {{const_cast<double *>(u_hin), D}});
    launch(k_bwd_h_cell<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c, g_h, h, u_hin,
                                                          da, g_rhs, dc, cot_hu, (int)overwrite);
    halo(pl, S(stream), {{cot_hu, D}});
    launch(k_bwd_h_gather<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c, cot_hu,
                                                            cu_out);
    PF_LAUNCH_CHECK("bwd_h_stage");
    return PF_OK;
  });
}

extern "C" int pf_bwd_momentum_outer(const pf_plan *plan, const double *y,
                                     const double *u_star, double *dc,
                                     void *stream) {
  PF_REQUIRE(plan && y && u_star && dc, "pf_bwd_momentum_outer: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream),
         {{const_cast<double *>(u_star), decltype(v)::kDim}});
    launch(k_bwd_mom_outer<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, y, u_star, dc);
    PF_LAUNCH_CHECK("bwd_momentum_outer");
    return PF_OK;
  });
}

extern "C" int pf_adj_momentum_rhs(const pf_plan *plan, const double *cot_rhs,
                                   const double *bc, double nu, double dt,
                                   double *du_n, double *dbc, double *dnu_dev,
                                   int32_t overwrite, void *workspace,
                                   void *stream) {
  PF_REQUIRE(plan && cot_rhs && du_n && dnu_dev && workspace,
             "pf_adj_momentum_rhs: null argument");
  const Plan &pl = P(plan);
  PF_REQUIRE((bc && dbc) || pl.d.m == 0, "pf_adj_momentum_rhs: null bc");
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    launch(k_adj_rhs_cells<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, cot_rhs, dt,
                                                             du_n, (int)overwrite);
    if (v.m > 0) {
      const int g = std::min(grid_for(v.m), pl.red_blocks);
      launch(k_adj_rhs_faces<decltype(v)>, g, kBlock, S(stream), 
          v, cot_rhs, bc, nu, dbc, dnu_dev, w.partials, w.counters);
    }
    PF_LAUNCH_CHECK("adj_momentum_rhs");
    return PF_OK;
  });
}

extern "C" int pf_adj_assemble_momentum(const pf_plan *plan, const double *dc,
                                        double nu, double *du_n,
                                        double *dnu_dev, void *workspace,
                                        void *stream) {
  PF_REQUIRE(plan && dc && du_n && dnu_dev && workspace,
             "pf_adj_assemble_momentum: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    const int g = std::min(grid_for(v.owned()), pl.red_blocks);
    halo(pl, S(stream),
         {{const_cast<double *>(dc), 2 * decltype(v)::kDim + 1}});
    launch(k_adj_assemble<decltype(v)>, g, kBlock, S(stream), v, dc, nu, du_n, dnu_dev,
                                                w.partials, w.counters);
    PF_LAUNCH_CHECK("adj_assemble_momentum");
    return PF_OK;
  });
}
