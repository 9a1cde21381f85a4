// forward.cu -- forward PISO building blocks (S/piso.py:123-460).
//
// One thread per cell, gathering over the 2d faces of its cell; neighbours
// come from index arithmetic (single block) or the packed neighbour table
// (multi-block).  Every kernel is a single streaming pass over SoA arrays.
#include "common.cuh"

namespace pf {

// -------------------------------------------------------------------------
// contravariant flux U^a = J (T u)_a   (S/piso.py:123-125)

template <class V>
__global__ void __launch_bounds__(kBlock) k_flux(V v,
                                                 const double *__restrict__ u,
                                                 double *__restrict__ flux) {
  constexpr int D = V::kDim;
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.n) return;
#pragma unroll
  for (int a = 0; a < D; ++a) flux[(int64_t)a * v.n + i] = v.flux(u, a, i);
}

// -------------------------------------------------------------------------
// momentum stencil C, rows normalised by J   (S/piso.py:293-319)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_assemble_momentum(V v, const double *__restrict__ flux,
                        double nu, double dt, double *__restrict__ c) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const auto cell = v.topo.cell(i);
  const double invj = v.IJ(i);
  double diag = 1.0 / dt;
  const int64_t n = v.n;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int a = f >> 1;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    const Face fc = v.topo.face(cell, f);
    double off = 0.0;
    if (fc.nb >= 0) {
      const double unb = flux[(int64_t)fc.ax * n + fc.nb];
      const double fmean = 0.5 * (flux[(int64_t)a * n + i] + (fc.neg ? -unb : unb));
      const double adv = 0.5 * nsgn * fmean * invj;
      const double visc = 0.5 * (nu * v.A(a, i) + nu * v.A(fc.ax, fc.nb)) * invj;
      off = adv - visc;
      diag += adv + visc;
    }
    c[(int64_t)(1 + f) * n + i] = off;
  }
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) {
      const int32_t e = fc.bidx;
      if ((__ldg(v.bface + e) >> 4) == PF_BKIND_DIRICHLET)
        diag += 2.0 * nu * __ldg(v.balpha + e) / v.J(i);
    }
  }
  c[i] = diag;
}

// -------------------------------------------------------------------------
// predictor right-hand side  (S/piso.py:356-372, orthogonal faces)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_momentum_rhs(V v, const double *__restrict__ u,
                   const double *__restrict__ bc,
                   const double *__restrict__ src, int src_uniform, double nu,
                   double dt, double *__restrict__ rhs) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  double r[D];
#pragma unroll
  for (int c = 0; c < D; ++c)
    r[c] = u[c * n + i] / dt + (src_uniform ? src[c] : src[c * n + i]);
  const double invj = v.IJ(i);
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb >= 0) continue;
    const int32_t e = fc.bidx;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    const double uflux = v.bflux(bc, e);
    double w;
    const bool dirichlet = (__ldg(v.bface + e) >> 4) == PF_BKIND_DIRICHLET;
    if (dirichlet)
      w = (2.0 * nu * __ldg(v.balpha + e) - uflux * nsgn) * invj;
    else
      w = -uflux * nsgn * invj;
#pragma unroll
    for (int c = 0; c < D; ++c) r[c] += bc[(int64_t)c * v.m + e] * w;
    if (dirichlet && v.finfo) {
      const FaceGeo g = face_geo(v, e);
      if (g.active) {
        double term[D];
        bcross_term(v, g, e, bc, term);
        const double sc = nsgn * nu / v.J(i);
#pragma unroll
        for (int c = 0; c < D; ++c) r[c] += term[c] * sc;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) rhs[c * n + i] = r[c];
}

// -------------------------------------------------------------------------
// K = -P, P the face-mean alpha_aa A^-1 operator  (S/piso.py:395-412)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_assemble_pressure(V v, const double *__restrict__ c, int c_is_a_inv,
                        double *__restrict__ k) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  const double ainv = c_is_a_inv ? c[i] : 1.0 / c[i];
  double diag = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int a = f >> 1;
    const Face fc = v.topo.face(cell, f);
    double off = 0.0;
    if (fc.nb >= 0) {
      // explicit roundings (no FMA contraction): the coupling is then the
      // same bits seen from either cell, P exactly symmetric
      // (T/test_piso.py:44-53)
      const double nbp = __dmul_rn(
          v.A(fc.ax, fc.nb), (c_is_a_inv ? c[fc.nb] : 1.0 / c[fc.nb]));
      const double pf = 0.5 * __dadd_rn(__dmul_rn(v.A(a, i), ainv), nbp);
      diag -= pf;
      off = -pf;
    }
    k[(int64_t)(1 + f) * n + i] = off;
  }
  k[i] = -diag;
}

// -------------------------------------------------------------------------
// h = A^-1 (rhs - H u)   (S/piso.py:608-612)

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_h_stage(V v, const double *__restrict__ c,
              const double *__restrict__ u, const double *__restrict__ rhs,
              double *__restrict__ h) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  double hu[D];
#pragma unroll
  for (int q = 0; q < D; ++q) hu[q] = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) continue;
    const double cf = c[(int64_t)(1 + f) * n + i];
#pragma unroll
    for (int q = 0; q < D; ++q) hu[q] += cf * u[q * n + fc.nb];
  }
  const double ainv = 1.0 / c[i];
#pragma unroll
  for (int q = 0; q < D; ++q) h[q * n + i] = ainv * (rhs[q * n + i] - hu[q]);
}

// -------------------------------------------------------------------------
// b = div_xi(h) with prescribed boundary fluxes  (S/piso.py:415-428)

template <class V>
__device__ __forceinline__ double cell_divergence(const V &v,
                                                  int32_t i,
                                                  const double *__restrict__ flux,
                                                  const double *__restrict__ bc) {
  constexpr int D = V::kDim;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  double b = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const int a = f >> 1;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    const Face fc = v.topo.face(cell, f);
    if (fc.nb >= 0) {
      const double unb = flux[(int64_t)fc.ax * n + fc.nb];
      b += nsgn * (0.5 * (flux[(int64_t)a * n + i] + (fc.neg ? -unb : unb)));
    }
  }
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) {
      const double nsgn = (f & 1) ? 1.0 : -1.0;
      b += nsgn * v.bflux(bc, fc.bidx);
    }
  }
  return b;
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_divergence_rhs(V v, const double *__restrict__ flux,
                     const double *__restrict__ bc, double *__restrict__ b) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  b[i] = cell_divergence(v, i, flux, bc);
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_divergence_max(V v, const double *__restrict__ flux,
                     const double *__restrict__ bc, double *partials,
                     unsigned *counter, double *out) {
  constexpr int D = V::kDim;
  double acc[1] = {0.0};
  RANGE_LOOP(i, v.rng())
    acc[0] = fmax(acc[0], fabs(cell_divergence(v, i, flux, bc) / v.J(i)));
  double tot[1];
  if (grid_reduce<1, true>(acc, partials, counter, tot)) *out = tot[0];
}

// -------------------------------------------------------------------------
// u = h - A^-1 T^t wide_grad(p, mirror)   (S/piso.py:452-455, 172-209)

template <class V>
__device__ __forceinline__ void mirror_grad(const V &v,
                                            const typename V::Cell &cell,
                                            const double *__restrict__ p,
                                            double (&g)[V::kDim]) {
  constexpr int D = V::kDim;
  const double pi = p[cell.i];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const Face lo = v.topo.face(cell, 2 * a);
    const Face hi = v.topo.face(cell, 2 * a + 1);
    const double vhi = hi.nb >= 0 ? p[hi.nb] : pi;
    const double vlo = lo.nb >= 0 ? p[lo.nb] : pi;
    g[a] = 0.5 * (vhi - vlo);
  }
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_correct_velocity(V v, const double *__restrict__ h,
                       const double *__restrict__ p,
                       const double *__restrict__ c, double *__restrict__ u) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  double g[D];
  mirror_grad(v, cell, p, g);
  const double ainv = 1.0 / c[i];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double e = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) e += v.T(j, k, i) * g[j];
    u[k * n + i] = h[k * n + i] - ainv * e;
  }
}

// -------------------------------------------------------------------------
// stencil matvec, plain and transposed (S/_kernels_c.pyx:52-63)

template <class V, bool kTrans>
__global__ void __launch_bounds__(kBlock)
    k_stencil_matvec(V v, const double *__restrict__ a, int ncomp,
                     const double *__restrict__ x, double *__restrict__ y) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  for (int q = 0; q < ncomp; ++q) {
    const double *xq = x + q * n;
    double acc = a[i] * xq[i];
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      const Face fc = v.topo.face(cell, f);
      if (fc.nb < 0) continue;
      const double coef = kTrans ? a[(int64_t)(1 + back_face(fc, f & 1)) * n + fc.nb]
                                 : a[(int64_t)(1 + f) * n + i];
      acc += coef * xq[fc.nb];
    }
    y[q * n + i] = acc;
  }
}

// -------------------------------------------------------------------------
// generic reductions

__global__ void __launch_bounds__(kBlock)
    k_reduce(const double *__restrict__ x, const double *__restrict__ y,
             int64_t len, int mode, double *partials, unsigned *counter,
             double *out) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (mode == 0) acc[0] += x[i];
    else if (mode == 1) acc[0] += x[i] * y[i];
    else acc[0] = fmax(acc[0], fabs(x[i]));
  }
  double tot[1];
  bool last = (mode == 2) ? grid_reduce<1, true>(acc, partials, counter, tot)
                          : grid_reduce<1, false>(acc, partials, counter, tot);
  if (last) *out = tot[0];
}

}  // namespace pf

// =========================================================================
// C ABI

using namespace pf;

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }
static const Plan &P(const pf_plan *p) {
  return *reinterpret_cast<const Plan *>(p);
}

#define PF_REQUIRE(cond, msg)        \
  do {                               \
    if (!(cond)) {                   \
      ::pf::set_error(msg);          \
      return PF_ERR_ARG;             \
    }                                \
  } while (0)

extern "C" int pf_contravariant_flux(const pf_plan *plan, const double *u,
                                     double *flux, void *stream) {
  PF_REQUIRE(plan && u && flux, "pf_contravariant_flux: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(u), decltype(v)::kDim}});
    launch(k_flux<decltype(v)>, grid_for(v.n), kBlock, S(stream), v, u, flux);
    PF_LAUNCH_CHECK("k_flux");
    return PF_OK;
  });
}

extern "C" int pf_assemble_momentum(const pf_plan *plan, const double *u_n,
                                    double nu, double dt, double *flux_scratch,
                                    double *c_out, void *stream) {
  PF_REQUIRE(plan && u_n && flux_scratch && c_out,
             "pf_assemble_momentum: null argument");
  return dispatch(P(plan), [&](auto v) {
    constexpr int D = decltype(v)::kDim;
    // slab plans: the face means need the neighbours' flux, so the flux is
    // formed on the ghost planes too (from exchanged velocities), and the
    // assembled stencil's ghost rows are exchanged for the transposed
    // gathers of the adjoint and the pressure assembly
    halo(P(plan), S(stream), {{const_cast<double *>(u_n), D}});
    launch(k_flux<decltype(v)>, grid_for(v.n), kBlock, S(stream), v, u_n, flux_scratch);
    launch(k_assemble_momentum<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), 
        v, flux_scratch, nu, dt, c_out);
    halo(P(plan), S(stream), {{c_out, 2 * D + 1}});
    PF_LAUNCH_CHECK("k_assemble_momentum");
    return PF_OK;
  });
}

extern "C" int pf_momentum_rhs(const pf_plan *plan, const double *u_n,
                               const double *bc, const double *source,
                               int32_t source_is_uniform, double nu, double dt,
                               double *rhs_out, void *stream) {
  PF_REQUIRE(plan && u_n && source && rhs_out, "pf_momentum_rhs: null argument");
  PF_REQUIRE(bc || P(plan).d.m == 0, "pf_momentum_rhs: null bc");
  return dispatch(P(plan), [&](auto v) {
    launch(k_momentum_rhs<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), 
        v, u_n, bc, source, source_is_uniform, nu, dt, rhs_out);
    PF_LAUNCH_CHECK("k_momentum_rhs");
    return PF_OK;
  });
}

extern "C" int pf_assemble_pressure(const pf_plan *plan, const double *c,
                                    int32_t c_is_a_inv, double *k_out,
                                    void *stream) {
  PF_REQUIRE(plan && c && k_out, "pf_assemble_pressure: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(c), 1}});
    launch(k_assemble_pressure<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c, c_is_a_inv,
                                                                 k_out);
    halo(P(plan), S(stream), {{k_out, 2 * decltype(v)::kDim + 1}});
    PF_LAUNCH_CHECK("k_assemble_pressure");
    return PF_OK;
  });
}

extern "C" int pf_h_stage(const pf_plan *plan, const double *c,
                          const double *u_cur, const double *rhs,
                          double *h_out, void *stream) {
  PF_REQUIRE(plan && c && u_cur && rhs && h_out, "pf_h_stage: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream),
         {{const_cast<double *>(u_cur), decltype(v)::kDim}});
    launch(k_h_stage<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, c, u_cur, rhs, h_out);
    PF_LAUNCH_CHECK("k_h_stage");
    return PF_OK;
  });
}

extern "C" int pf_divergence_rhs(const pf_plan *plan, const double *h,
                                 const double *bc, double *flux_scratch,
                                 double *b_out, void *stream) {
  PF_REQUIRE(plan && h && flux_scratch && b_out,
             "pf_divergence_rhs: null argument");
  PF_REQUIRE(bc || P(plan).d.m == 0, "pf_divergence_rhs: null bc");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(h), decltype(v)::kDim}});
    launch(k_flux<decltype(v)>, grid_for(v.n), kBlock, S(stream), v, h, flux_scratch);
    launch(k_divergence_rhs<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), 
        v, flux_scratch, bc, b_out);
    PF_LAUNCH_CHECK("k_divergence_rhs");
    return PF_OK;
  });
}

extern "C" int pf_correct_velocity(const pf_plan *plan, const double *h,
                                   const double *p, const double *c,
                                   double *u_out, void *stream) {
  PF_REQUIRE(plan && h && p && c && u_out, "pf_correct_velocity: null argument");
  return dispatch(P(plan), [&](auto v) {
    halo(P(plan), S(stream), {{const_cast<double *>(p), 1}});
    launch(k_correct_velocity<decltype(v)>, grid_for(v.owned()), kBlock, S(stream), v, h, p, c,
                                                                 u_out);
    PF_LAUNCH_CHECK("k_correct_velocity");
    return PF_OK;
  });
}

static int red_grid(const Plan &p, int64_t len) {
  int g = grid_for(len);
  return g < p.red_blocks ? g : p.red_blocks;
}

extern "C" int pf_divergence_max(const pf_plan *plan, const double *u,
                                 const double *bc, double *flux_scratch,
                                 void *workspace, double *out_host,
                                 void *stream) {
  PF_REQUIRE(plan && u && flux_scratch && workspace && out_host,
             "pf_divergence_max: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  int rc = dispatch(pl, [&](auto v) {
    halo(pl, S(stream), {{const_cast<double *>(u), decltype(v)::kDim}});
    launch(k_flux<decltype(v)>, grid_for(v.n), kBlock, S(stream), v, u, flux_scratch);
    launch(k_divergence_max<decltype(v)>, red_grid(pl, v.owned()), kBlock,
           S(stream), v, flux_scratch, bc, w.partials, w.counters, w.scalars);
    PF_LAUNCH_CHECK("k_divergence_max");
    return PF_OK;
  });
  if (rc) return rc;
  return d2h(pl, out_host, w.scalars, sizeof(double), S(stream));
}

// the same into a device scalar, without waiting: the step's diagnostics
// read it when asked, so no host round trip sits between the forward step
// and the adjoint
extern "C" int pf_divergence_max_dev(const pf_plan *plan, const double *u,
                                     const double *bc, double *flux_scratch,
                                     void *workspace, double *out_dev,
                                     void *stream) {
  PF_REQUIRE(plan && u && flux_scratch && workspace && out_dev,
             "pf_divergence_max_dev: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  int rc = dispatch(pl, [&](auto v) {
    halo(pl, S(stream), {{const_cast<double *>(u), decltype(v)::kDim}});
    launch(k_flux<decltype(v)>, grid_for(v.n), kBlock, S(stream), v, u, flux_scratch);
    launch(k_divergence_max<decltype(v)>, red_grid(pl, v.owned()), kBlock,
           S(stream), v, flux_scratch, bc, w.partials, w.counters, w.scalars);
    PF_LAUNCH_CHECK("k_divergence_max");
    return PF_OK;
  });
  if (rc) return rc;
  PF_CUDA(cudaMemcpyAsync(out_dev, w.scalars, sizeof(double),
                          cudaMemcpyDeviceToDevice, S(stream)));
  return PF_OK;
}

// ---------------------------------------------------------------------------
// channel drivers (S/piso.py:512-546): adaptive_dt's CFL peak and the
// per-step wall forcing, each one fused reduction

namespace pf {

// max over owned cells of sum_a |U^a| / J (adaptive_dt, S/piso.py:512-520)
template <class V>
__global__ void __launch_bounds__(kBlock)
    k_cfl_peak(V v, const double *__restrict__ u, double *partials,
               unsigned *counter, double *out) {
  constexpr int D = V::kDim;
  double acc[1] = {0.0};
  RANGE_LOOP(i, v.rng()) {
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) r += fabs(v.flux(u, a, i));
    acc[0] = fmax(acc[0], r / v.J(i));
  }
  double tot[1];
  if (grid_reduce<1, true>(acc, partials, counter, tot)) *out = tot[0];
}

constexpr int kMaxWalls = 8;

// wall_shear_mean / wall_forcing_source (S/piso.py:523-542): per wall w the
// mean of u[c, flow] / dist over its first cell row (sum / cnt[w]: on slab
// plans the sums span the ranks, cnt is the global row size), then
// source[flow] = nu mean_w |mean_w| / delta, the other components 0
__global__ void __launch_bounds__(kBlock)
    k_wall_forcing(const double *__restrict__ u, int64_t n, int flow, int d,
                   const int32_t *__restrict__ cells,
                   const double *__restrict__ dist, const int32_t *seg,
                   const double *cnt, int nwall, double nu, double delta,
                   double *out,
                   double *partials, unsigned *counter) {
  double acc[kMaxWalls];
#pragma unroll
  for (int k = 0; k < kMaxWalls; ++k) acc[k] = 0.0;
  const int32_t m = seg[nwall];
  for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += gridDim.x * blockDim.x) {
    int w = 0;
    while (w + 1 < nwall && e >= seg[w + 1]) ++w;
    const double val = u[flow * n + cells[e]] / dist[e];
#pragma unroll
    for (int k = 0; k < kMaxWalls; ++k)
      if (k == w) acc[k] += val;
  }
  double tot[kMaxWalls];
  if (grid_reduce<kMaxWalls>(acc, partials, counter, tot)) {
    double sh = 0.0;
    for (int w = 0; w < nwall; ++w)
      sh += fabs(tot[w] / cnt[w]);
    sh /= nwall;
    for (int c = 0; c < d; ++c) out[c] = c == flow ? nu * sh / delta : 0.0;
  }
}

}  // namespace pf

extern "C" int pf_cfl_peak(const pf_plan *plan, const double *u,
                           void *workspace, double *out_dev, void *stream) {
  PF_REQUIRE(plan && u && workspace && out_dev, "pf_cfl_peak: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  return dispatch(pl, [&](auto v) {
    launch(k_cfl_peak<decltype(v)>, red_grid(pl, v.owned()), kBlock,
           S(stream), v, u, w.partials, w.counters, out_dev);
    PF_LAUNCH_CHECK("k_cfl_peak");
    return PF_OK;
  });
}

extern "C" int pf_wall_forcing(const pf_plan *plan, const double *u,
                               int32_t flow_axis, const int32_t *cells,
                               const double *dist, const int32_t *seg,
                               const double *cnt, int32_t nwall, int32_t m,
                               double nu,
                               double delta, double *out_dev, void *workspace,
                               void *stream) {
  PF_REQUIRE(plan && u && cells && dist && seg && cnt && out_dev && workspace &&
                 nwall >= 1 && nwall <= kMaxWalls && m >= 1,
             "pf_wall_forcing: bad argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  launch(k_wall_forcing, red_grid(pl, m), kBlock, S(stream), u, pl.d.n,
         (int)flow_axis, (int)pl.d.dim, cells, dist, seg, cnt, (int)nwall, nu,
         delta, out_dev, w.partials, w.counters);
  PF_LAUNCH_CHECK("k_wall_forcing");
  return PF_OK;
}

extern "C" int pf_stencil_matvec(const pf_plan *plan, const double *a,
                                 int32_t transpose, int32_t ncomp,
                                 const double *x, double *y, void *stream) {
  PF_REQUIRE(plan && a && x && y && ncomp >= 1, "pf_stencil_matvec: bad argument");
  return dispatch(P(plan), [&](auto v) {
    using V = decltype(v);
    halo(P(plan), S(stream), {{const_cast<double *>(x), ncomp}});
    if (transpose)
      halo(P(plan), S(stream), {{const_cast<double *>(a), 2 * V::kDim + 1}});
    if (transpose)
      launch(k_stencil_matvec<V, true>, grid_for(v.owned()), kBlock, S(stream), v, a, ncomp, x, y);
    else
      launch(k_stencil_matvec<V, false>, grid_for(v.owned()), kBlock, S(stream), v, a, ncomp, x, y);
    PF_LAUNCH_CHECK("k_stencil_matvec");
    return PF_OK;
  });
}

static int reduce_common(const pf_plan *plan, const double *x, const double *y,
                         int64_t len, int mode, void *workspace,
                         double *out_host, void *stream) {
  PF_REQUIRE(plan && x && workspace && out_host, "pf_reduce: null argument");
  const Plan &pl = P(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  launch(k_reduce, red_grid(pl, len), kBlock, S(stream), x, y, len, mode,
         w.partials, w.counters, w.scalars);
  PF_LAUNCH_CHECK("k_reduce");
  return d2h(pl, out_host, w.scalars, sizeof(double), S(stream));
}

extern "C" int pf_reduce_sum(const pf_plan *plan, const double *x, int64_t len,
                             void *workspace, double *out_host, void *stream) {
  return reduce_common(plan, x, nullptr, len, 0, workspace, out_host, stream);
}
extern "C" int pf_reduce_dot(const pf_plan *plan, const double *x,
                             const double *y, int64_t len, void *workspace,
                             double *out_host, void *stream) {
  PF_REQUIRE(y, "pf_reduce_dot: null argument");
  return reduce_common(plan, x, y, len, 1, workspace, out_host, stream);
}
extern "C" int pf_reduce_maxabs(const pf_plan *plan, const double *x,
                                int64_t len, void *workspace, double *out_host,
                                void *stream) {
  return reduce_common(plan, x, nullptr, len, 2, workspace, out_host, stream);
}
