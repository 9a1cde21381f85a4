// boundary.cu -- advective outflow preprocessing (S/piso.py:467-509).
//
// Runs before the differentiated part of the step: outflow-face velocities
// are relaxed towards the adjacent cell values, then rescaled so the net
// boundary volume flux vanishes (or seeded with a uniform normal outflow on a
// cold start).  Two passes over the m boundary entries; the decision between
// "rescale", "cold seed" and "leave" is taken in the last CTA of the first
// pass and read by the second.
#include <algorithm>

#include "common.cuh"

namespace pf {

struct OutflowState {
  double fixed, out_total, area, scale, cold_c;
  int32_t mode;  // 0 leave, 1 rescale, 2 cold seed
  int32_t pad;
};

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_outflow_relax(V v, const double *__restrict__ u, double *__restrict__ bc,
                    double dt, OutflowState *st, double *partials,
                    unsigned *counter) {
  constexpr int D = V::kDim;
  const int64_t n = v.n, m = v.m;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < v.m;
       e += gridDim.x * blockDim.x) {
    // slab plans: entries of ghost-plane cells belong to a neighbour rank
    const int32_t ie = __ldg(v.bcell + e);
    if (ie < v.i0 || ie >= v.i1) continue;
    const int bf = __ldg(v.bface + e);
    const int f = bf & 15, kind = bf >> 4;
    const double nsgn = (f & 1) ? 1.0 : -1.0;
    if (kind == PF_BKIND_DIRICHLET) {
      acc[0] += nsgn * v.bflux(bc, e);
      continue;
    }
    const int32_t i = __ldg(v.bcell + e);
    double speed = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j)
      speed += __ldg(v.bt + j * m + e) * bc[j * m + e];
    const double a = fmax(2.0 * dt * speed * nsgn, 0.0);
#pragma unroll
    for (int j = 0; j < D; ++j)
      bc[j * m + e] = (bc[j * m + e] + a * u[j * n + i]) / (1.0 + a);
    acc[1] += nsgn * v.bflux(bc, e);
    acc[2] += __ldg(v.bjac + e);
  }
  double tot[3];
  if (grid_reduce<3>(acc, partials, counter, tot)) {
    st->fixed = tot[0];
    st->out_total = tot[1];
    st->area = tot[2];
    st->scale = 1.0;
    if (fabs(tot[1]) < 1e-13 * fmax(1.0, fabs(tot[0]))) {
      if (fabs(tot[0]) <= 1e-12) {
        st->mode = 0;
      } else {
        st->mode = 2;
        st->cold_c = -tot[0] / tot[2];
      }
    } else {
      st->mode = 1;
      st->scale = -tot[0] / tot[1];
    }
  }
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_outflow_apply(V v, double *__restrict__ bc, const OutflowState *st) {
  constexpr int D = V::kDim;
  const int64_t m = v.m;
  const int mode = st->mode;
  if (mode == 0) return;
  const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v.m) return;
  const int bf = __ldg(v.bface + e);
  if ((bf >> 4) != PF_BKIND_OUTFLOW) return;
  if (mode == 1) {
    const double s = st->scale;
#pragma unroll
    for (int j = 0; j < D; ++j) bc[j * m + e] = bc[j * m + e] * s;
  } else {
    const double nsgn = (bf & 1) ? 1.0 : -1.0;
    double tt = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double t = __ldg(v.bt + j * m + e);
      tt += t * t;
    }
#pragma unroll
    for (int j = 0; j < D; ++j)
      bc[j * m + e] = st->cold_c * nsgn * (__ldg(v.bt + j * m + e) / tt);
  }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_advective_outflow_update(const pf_plan *plan,
                                           const double *u, double *bc_inout,
                                           double dt, void *workspace,
                                           double *scale_host, void *stream) {
  if (!plan || !u || !bc_inout || !workspace || !scale_host) {
    set_error("pf_advective_outflow_update: null argument");
    return PF_ERR_ARG;
  }
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  Workspace w = carve(workspace, pl.d.n, pl.d.dim);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  OutflowState *st = reinterpret_cast<OutflowState *>(w.scalars);
  if (pl.d.m == 0) {
    *scale_host = 1.0;
    return PF_OK;
  }
  int rc = dispatch(pl, [&](auto v) {
    const int g = std::min(grid_for(v.m), pl.red_blocks);
    launch(k_outflow_relax<decltype(v)>, g, kBlock, s, v, u, bc_inout, dt, st, w.partials,
                                         w.counters);
    launch(k_outflow_apply<decltype(v)>, grid_for(v.m), kBlock, s, v, bc_inout, st);
    PF_LAUNCH_CHECK("advective_outflow_update");
    return PF_OK;
  });
  if (rc) return rc;
  OutflowState hs;
  rc = d2h(pl, &hs, st, sizeof(hs), s);
  if (rc) return rc;
  *scale_host = hs.scale;
  return PF_OK;
}
