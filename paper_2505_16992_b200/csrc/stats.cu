// stats.cu -- wall-normal slice statistics of a channel velocity field
// (S/stats.py:234-290): per-slice means and central co-moments over the
// homogeneous planes, and the cotangent of (mean, covariance) back onto the
// velocity -- the statistics loss of the LES training runs,
// evaluated on the device.
//
// A slice is one index of the wall axis (axis 1 of a 3D / axis 0 of a 2D
// box); its cells are the (x, z) planes of the owned range.  Two passes:
// sums -> means, then central products around those means (the reference's
// two-pass form, so no cancellation).  Each pass reduces (slice, X-chunk)
// blocks into partials that one small kernel folds in a fixed order; slab
// plans then add the ranks' sums (comm_vec_allreduce).  No float atomics:
// the result is bitwise reproducible.
#include "common.cuh"

namespace pf {

constexpr int kStatK = 16;     // values per slice: 3 sums / 6 co-moments +
                               // 3 third + 3 fourth moments (3D)
constexpr int kStatXC = 16;    // X planes per block

struct SliceGeo {
  int32_t nx, ny, nz;   // slices = ny; homogeneous (nx owned, nz)
  int32_t x0;           // first owned plane (slab ghost offset)
  int32_t xb;           // X blocks
  int32_t dim;          // 2 or 3
  int64_t n;            // component stride
  int64_t sx, sy;       // strides of the X and wall axes
  double count;         // cells per slice over all ranks
};

// pass 0: sums u_c; pass 1: central products c_i c_j (i <= j) and the
// third / fourth single-channel central moments
template <int PASS>
__global__ void __launch_bounds__(kBlock)
    k_slice_partial(SliceGeo g, const double *__restrict__ u,
                    const double *__restrict__ mean,
                    double *__restrict__ part) {
  const int y = blockIdx.y, xb = blockIdx.x;
  const int D = g.dim;
  double acc[kStatK];
#pragma unroll
  for (int k = 0; k < kStatK; ++k) acc[k] = 0.0;
  double mu[3] = {0.0, 0.0, 0.0};
  if (PASS == 1)
    for (int c = 0; c < D; ++c) mu[c] = mean[y * D + c];
  const int32_t xs = xb * kStatXC, xe = min(xs + kStatXC, g.nx);
  const int64_t cells = (int64_t)(xe - xs) * g.nz;
  for (int64_t t = threadIdx.x; t < cells; t += blockDim.x) {
    const int32_t x = g.x0 + xs + (int32_t)(t / g.nz);
    const int32_t z = (int32_t)(t % g.nz);
    const int64_t i = (int64_t)x * g.sx + (int64_t)y * g.sy + z;
    double v[3];
    for (int c = 0; c < 3; ++c) v[c] = c < D ? u[c * g.n + i] - mu[c] : 0.0;
    if (PASS == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += v[c];
    } else {
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) acc[k++] += v[a] * v[b];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double v2 = v[c] * v[c];
        acc[6 + c] += v2 * v[c];
        acc[9 + c] += v2 * v2;
      }
    }
  }
  block_reduce<kStatK>(acc);
  if (threadIdx.x == 0) {
    double *o = part + ((int64_t)y * g.xb + xb) * kStatK;
#pragma unroll
    for (int k = 0; k < kStatK; ++k) o[k] = acc[k];
  }
}

// fold the X blocks of every (slice, value) in block order
__global__ void __launch_bounds__(kBlock)
    k_slice_fold(SliceGeo g, const double *__restrict__ part,
                 double *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.ny * kStatK) return;
  const int y = t / kStatK, k = t % kStatK;
  double s = 0.0;
  for (int b = 0; b < g.xb; ++b) s += part[((int64_t)y * g.xb + b) * kStatK + k];
  out[t] = s;
}

// sums -> means (in place on the first D values of every slice row)
__global__ void k_slice_means(SliceGeo g, const double *__restrict__ sums,
                              double *__restrict__ mean) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.ny * g.dim) return;
  const int y = t / g.dim, c = t % g.dim;
  mean[t] = sums[y * kStatK + c] / g.count;
}

// co-moment sums -> covariance (Y, D, D) and third / fourth moments (Y, D)
__global__ void k_slice_cov(SliceGeo g, const double *__restrict__ sums,
                            double *__restrict__ cov, double *__restrict__ m3,
                            double *__restrict__ m4) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= g.ny) return;
  const int D = g.dim;
  const double *s = sums + (int64_t)y * kStatK;
  int k = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b, ++k) {
      if (a >= D || b >= D) continue;
      const double v = s[k] / g.count;
      cov[((int64_t)y * D + a) * D + b] = v;
      cov[((int64_t)y * D + b) * D + a] = v;
    }
  for (int c = 0; c < D; ++c) {
    if (m3) m3[y * D + c] = s[6 + c] / g.count;
    if (m4) m4[y * D + c] = s[9 + c] / g.count;
  }
}

// du_i = (sym(d_cov) . (u_i - mean) + d_mean) / count on the owned cells
// (frame_profile_backward, S/stats.py:281-290)
__global__ void __launch_bounds__(kBlock)
    k_slice_backward(SliceGeo g, const double *__restrict__ u,
                     const double *__restrict__ mean,
                     const double *__restrict__ dmean,
                     const double *__restrict__ dcov,
                     double *__restrict__ du) {
  const int64_t cells = (int64_t)g.nx * g.ny * g.nz;
  const int D = g.dim;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cells;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t z = (int32_t)(t % g.nz);
    const int64_t r = t / g.nz;
    const int32_t y = (int32_t)(r % g.ny);
    const int32_t x = g.x0 + (int32_t)(r / g.ny);
    const int64_t i = (int64_t)x * g.sx + (int64_t)y * g.sy + z;
    double cen[3];
    for (int c = 0; c < D; ++c) cen[c] = u[c * g.n + i] - mean[y * D + c];
    for (int a = 0; a < D; ++a) {
      double s = dmean[y * D + a];
      for (int b = 0; b < D; ++b) {
        const double sym = dcov[((int64_t)y * D + a) * D + b] +
                           dcov[((int64_t)y * D + b) * D + a];
        s += sym * cen[b];
      }
      du[a * g.n + i] = s / g.count;
    }
  }
}

static int slice_geo(const Plan &p, int wall_axis, SliceGeo &g) {
  if (p.d.topo != PF_TOPO_BOX) {
    set_error("slice statistics need a single-block box plan");
    return PF_ERR_UNSUPPORTED;
  }
  const int D = p.d.dim;
  const int wa = wall_axis;
  if ((D == 3 && wa != 1) || (D == 2 && wa != 0 && wa != 1)) {
    set_error("slice statistics: wall axis must be 1 (3D) or 0 / 1 (2D)");
    return PF_ERR_UNSUPPORTED;
  }
  g.dim = D;
  g.n = p.d.n;
  const int64_t plane = p.slab ? p.plane : 0;
  if (D == 3) {
    g.ny = (int32_t)p.d.box_shape[1];
    g.nz = (int32_t)p.d.box_shape[2];
    g.sy = g.nz;
    g.sx = (int64_t)g.ny * g.nz;
    g.x0 = p.slab ? 1 : 0;
    g.nx = p.slab ? (int32_t)p.nxl : (int32_t)p.d.box_shape[0];
    g.count = (double)(p.slab ? p.d.slab_nx : g.nx) * g.nz;
  } else if (wa == 1) {
    // 2D, slices along axis 1: "x" = axis 0, "z" absent
    g.ny = (int32_t)p.d.box_shape[1];
    g.nz = 1;
    g.sy = 1;
    g.sx = g.ny;
    g.x0 = p.slab ? 1 : 0;
    g.nx = p.slab ? (int32_t)p.nxl : (int32_t)p.d.box_shape[0];
    g.count = (double)(p.slab ? p.d.slab_nx : g.nx);
  } else {
    // 2D, slices along axis 0: the homogeneous axis is 1 ("z")
    if (p.slab) {
      set_error("slice statistics: slab plans slice along axis 1");
      return PF_ERR_UNSUPPORTED;
    }
    g.ny = (int32_t)p.d.box_shape[0];
    g.nz = (int32_t)p.d.box_shape[1];
    g.sy = g.nz;
    g.sx = 0;
    g.x0 = 0;
    g.nx = 1;
    g.count = (double)g.nz;
  }
  (void)plane;
  g.xb = (g.nx + kStatXC - 1) / kStatXC;
  if ((int64_t)g.ny * g.xb * kStatK > (int64_t)kWsVectors * D * p.d.n) {
    set_error("slice statistics: workspace too small");
    return PF_ERR_ARG;
  }
  return PF_OK;
}

}  // namespace pf

using namespace pf;

extern "C" int pf_slice_moments(const pf_plan *plan, const double *u,
                                int32_t wall_axis, double *mean, double *cov,
                                double *m3, double *m4, void *workspace,
                                void *stream) {
  if (!plan || !u || !mean || !cov || !workspace) {
    set_error("pf_slice_moments: null argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  SliceGeo g;
  int rc = slice_geo(p, wall_axis, g);
  if (rc) return rc;
  Workspace w = carve(workspace, p.d.n, p.d.dim);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *part = w.vecs;
  double *sums = w.vecs + (int64_t)g.ny * g.xb * kStatK;
  const dim3 grid(g.xb, g.ny);
  const int nv = g.ny * kStatK;
  launch(k_slice_partial<0>, grid, kBlock, s, g, u,
         (const double *)nullptr, part);
  launch(k_slice_fold, grid_for(nv), kBlock, s, g, (const double *)part, sums);
  rc = comm_vec_allreduce_n(p, sums, nv, 0, s);
  if (rc) return rc;
  launch(k_slice_means, grid_for(g.ny * g.dim), kBlock, s, g,
         (const double *)sums, mean);
  launch(k_slice_partial<1>, grid, kBlock, s, g, u, (const double *)mean,
         part);
  launch(k_slice_fold, grid_for(nv), kBlock, s, g, (const double *)part, sums);
  rc = comm_vec_allreduce_n(p, sums, nv, 0, s);
  if (rc) return rc;
  launch(k_slice_cov, grid_for(g.ny), kBlock, s, g, (const double *)sums, cov,
         m3, m4);
  PF_LAUNCH_CHECK("pf_slice_moments");
  return PF_OK;
}

extern "C" int pf_slice_moments_backward(const pf_plan *plan, const double *u,
                                         int32_t wall_axis, const double *mean,
                                         const double *d_mean,
                                         const double *d_cov, double *du,
                                         void *stream) {
  if (!plan || !u || !mean || !d_mean || !d_cov || !du) {
    set_error("pf_slice_moments_backward: null argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  SliceGeo g;
  int rc = slice_geo(p, wall_axis, g);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t cells = (int64_t)g.nx * g.ny * g.nz;
  launch(k_slice_backward, (int)std::min<int64_t>(grid_for(cells),
                                                  p.num_sms * 16),
         kBlock, s, g, u, mean, d_mean, d_cov, du);
  PF_LAUNCH_CHECK("pf_slice_moments_backward");
  return PF_OK;
}
