// mg.cu -- geometric multigrid V(1,1) preconditioner (see mg.cuh).
//
// Level layout: canonical (X, Y, Z) C-order, index ((x*sy)+y)*sz+z, so the
// Y lines of the smoother are strided by sz and threads of a warp take
// consecutive z -- every line-solve load is coalesced across the warp.
#include <algorithm>
#include <mutex>

#include "cgstate.cuh"
#include "mg.cuh"
#include "spectral.cuh"

namespace pf {

constexpr int kLineBlock = 128;
constexpr int kChunk = 8;  // rows batched per load phase of a line sweep

__device__ __forceinline__ int32_t lid(const MgLevel &L, int32_t x, int32_t y,
                                       int32_t z) {
  return (x * L.sy + y) * L.sz + z;
}

// parent (coarse) index; coarsening factors are 1 or 2: shifts, no division
__device__ __forceinline__ int32_t parent(const MgLevel &F, const MgLevel &C,
                                          int32_t x, int32_t y, int32_t z) {
  return ((x >> (F.fx - 1)) * C.sy + (y >> (F.fy - 1))) * C.sz +
         (z >> (F.fz - 1));
}

#define MG_DONE_RETURN \
  if (done && *done) return

// ---------------------------------------------------------------------------
// setup

// level-0 face weights from the K stencil (row 1 + 2a + 1 holds -w)
__global__ void __launch_bounds__(kBlock)
    k_mg_faces0(MgLevel L, const double *__restrict__ k, int64_t n, int ax0,
                int ax1, int ax2, const int *done) {
  MG_DONE_RETURN;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  L.wx[i] = ax0 >= 0 ? -k[(int64_t)(2 + 2 * ax0) * n + i] : 0.0;
  L.wy[i] = -k[(int64_t)(2 + 2 * ax1) * n + i];
  L.wz[i] = ax2 >= 0 ? -k[(int64_t)(2 + 2 * ax2) * n + i] : 0.0;
}

// coarse face = sum of the fine faces crossing it
__global__ void __launch_bounds__(kBlock)
    k_mg_aggregate(MgLevel F, MgLevel C, const int *done) {
  MG_DONE_RETURN;
  const int32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= C.n) return;
  const Cell3 c = decode(C, I);
  double wx = 0.0, wy = 0.0, wz = 0.0;
  for (int dx = 0; dx < F.fx; ++dx)
    for (int dy = 0; dy < F.fy; ++dy)
      for (int dz = 0; dz < F.fz; ++dz) {
        const int32_t j = lid(F, F.fx * c.x + dx, F.fy * c.y + dy,
                              F.fz * c.z + dz);
        if (dx == F.fx - 1) wx += F.wx[j];
        if (dy == F.fy - 1) wy += F.wy[j];
        if (dz == F.fz - 1) wz += F.wz[j];
      }
  C.wx[I] = C.sx > 1 ? wx : 0.0;  // a 1-wide periodic axis: self loop
  C.wy[I] = wy;
  C.wz[I] = C.sz > 1 ? wz : 0.0;
}

// Thomas factors of the Y-line matrices (diagonal = sum of the 6 faces)
__global__ void __launch_bounds__(kBlock)
    k_mg_factor(MgLevel L, const int *done) {
  MG_DONE_RETURN;
  const int32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L.sx * L.sz) return;
  const int32_t x = l / L.sz, z = l % L.sz;
  double cprev = 0.0, wprev = 0.0;
  for (int y = 0; y < L.sy; ++y) {
    Cell3 c;
    c.x = x;
    c.y = y;
    c.z = z;
    c.i = lid(L, x, y, z);
    if (L.pinned && y == L.sy - 1) {
      L.ivd[c.i] = 1.0;
      L.cp[c.i] = 0.0;
      break;
    }
    const Nbhd b = nbhd(L, c);
    const double d = b.wxp + b.wxm + b.wyp + b.wym + b.wzp + b.wzm;
    const double iv = 1.0 / (d + wprev * cprev);
    const double cc = -b.wyp * iv;
    L.ivd[c.i] = iv;
    L.cp[c.i] = cc;
    cprev = cc;
    wprev = b.wyp;
  }
}

// ---------------------------------------------------------------------------
// line smoothing
//
// Y-line solve T z = rhs for the line (x, z), loads batched kChunk rows at a
// time so the serial recurrence never waits on one load per row.  `tmp`
// holds the forward sweep and may alias rhs (each element is read before it
// is overwritten).  mode 0: out = w z;  mode 2: out += P x_c + w z (the
// coarse correction prolonged on the fly).  kSums: accumulate the CG z-sums
// (sum z, sum r.z, sum r, with r = L.r) of the written values.
template <int kMode, bool kSums = false>
__device__ __forceinline__ void line_solve(const MgLevel &L, int32_t x,
                                           int32_t z, const double *rhs,
                                           double *tmp, double *out,
                                           double omega,
                                           const MgLevel *C = nullptr,
                                           double *sums = nullptr) {
  const int32_t st = L.sz;
  const int32_t base = lid(L, x, 0, z);
  const int32_t sy = L.sy;
  double dp = 0.0, wprev = 0.0;
  for (int y0 = 0; y0 < sy; y0 += kChunk) {
    double rr[kChunk], iv[kChunk], ww[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const int y = y0 + k;
      if (y < sy) {
        const int32_t i = base + y * st;
        rr[k] = rhs[i];
        iv[k] = L.ivd[i];
        ww[k] = L.wy[i];
      }
    }
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const int y = y0 + k;
      if (y < sy) {
        dp = (L.pinned && y == sy - 1) ? 0.0 : (rr[k] + wprev * dp) * iv[k];
        wprev = ww[k];
        tmp[base + y * st] = dp;
      }
    }
  }
  int32_t cbase = 0, cst = 0;
  if (kMode == 2) {
    cbase = lid(*C, x >> (L.fx - 1), 0, z >> (L.fz - 1));
    cst = C->sz;
  }
  double znext = 0.0;
  for (int y0 = sy - 1; y0 >= 0; y0 -= kChunk) {
    double tt[kChunk], cc[kChunk], oo[kChunk], rr[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const int y = y0 - k;
      if (y >= 0) {
        const int32_t i = base + y * st;
        tt[k] = tmp[i];
        cc[k] = L.cp[i];
        if (kMode == 2) oo[k] = out[i] + C->x[cbase + (y >> (L.fy - 1)) * cst];
        if (kSums) rr[k] = L.r[i];
      }
    }
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const int y = y0 - k;
      if (y >= 0) {
        const double zv = tt[k] - cc[k] * znext;
        znext = zv;
        const double o = kMode == 0 ? omega * zv : oo[k] + omega * zv;
        out[base + y * st] = o;
        if (kSums) {
          sums[0] += o;
          sums[1] += rr[k] * o;
          sums[2] += rr[k];
        }
      }
    }
  }
}

// x = omega T^-1 r over every line
__global__ void __launch_bounds__(kLineBlock)
    k_mg_smooth0(MgLevel L, const double *__restrict__ r, double *x,
                 double omega, const int *done) {
  MG_DONE_RETURN;
  const int32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L.sx * L.sz) return;
  line_solve<0>(L, l / L.sz, l % L.sz, r, x, x, omega);
}

// x += P x_c + omega T^-1 res  (res = r - K (x + P x_c), consumed)
__global__ void __launch_bounds__(kLineBlock)
    k_mg_smooth2(MgLevel L, double *res, double *x, double omega, MgLevel C,
                 const int *done) {
  MG_DONE_RETURN;
  const int32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L.sx * L.sz) return;
  line_solve<2>(L, l / L.sz, l % L.sz, res, res, x, omega, &C);
}

// level 0 of the CG's V-cycle: the final smoothing pass also accumulates the
// CG z-sums and evaluates beta (k_cg_zsum folded in); grid-stride over lines
// so the grid fits the reduction partials
__global__ void __launch_bounds__(kLineBlock)
    k_mg_smooth2_cg(MgLevel L, double *res, double *x, double omega,
                    MgLevel C, CgFuse fz, const int *done) {
  MG_DONE_RETURN;
  double sums[3] = {0.0, 0.0, 0.0};
  for (int32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < L.sx * L.sz;
       l += gridDim.x * blockDim.x)
    line_solve<2, true>(L, l / L.sz, l % L.sz, res, res, x, omega, &C, sums);
  double tot[3];
  if (grid_reduce<3>(sums, fz.partials, fz.counter, tot))
    cg_fin_z(fz.st, tot[0], tot[1], tot[2], (int32_t)L.n, fz.initial != 0);
}

// ---------------------------------------------------------------------------
// residual transfer

// coarse rhs = sum over the aggregate of r - K x, coarse cell I
__device__ __forceinline__ void resid_restrict_at(const MgLevel &F,
                                                  const double *r,
                                                  const double *x,
                                                  const MgLevel &C,
                                                  int32_t I, double corr) {
  const Cell3 cc = decode(C, I);
  double acc = 0.0;
  for (int dx = 0; dx < F.fx; ++dx)
    for (int dy = 0; dy < F.fy; ++dy)
      for (int dz = 0; dz < F.fz; ++dz) {
        Cell3 c;
        c.x = F.fx * cc.x + dx;
        c.y = F.fy * cc.y + dy;
        c.z = F.fz * cc.z + dz;
        c.i = lid(F, c.x, c.y, c.z);
        const Nbhd b = nbhd(F, c);
        acc += r[c.i] - kx(b, c.i, x);
      }
  C.r[I] = corr * acc;
}

__global__ void __launch_bounds__(kBlock)
    k_mg_resid_restrict(MgLevel F, const double *__restrict__ r,
                        const double *__restrict__ x, MgLevel C,
                        double corr, const int *done) {
  MG_DONE_RETURN;
  const int32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= C.n) return;
  resid_restrict_at(F, r, x, C, I, corr);
}

// res = r - K (x + P x_c) at fine cell i: prolongation fused into the
// residual; x itself is updated by the following smoothing pass, so no
// thread writes what another thread reads
__device__ __forceinline__ void prolong_resid_at(const MgLevel &F,
                                                 const double *r,
                                                 const double *x, double *res,
                                                 const MgLevel &C, int32_t i) {
  const Cell3 c = decode(F, i);
  const Nbhd b = nbhd(F, c);
  const double *cxv = C.x;
  const int32_t xp = c.x + 1 < F.sx ? c.x + 1 : 0;
  const int32_t xm = c.x > 0 ? c.x - 1 : F.sx - 1;
  const int32_t zp = c.z + 1 < F.sz ? c.z + 1 : 0;
  const int32_t zm = c.z > 0 ? c.z - 1 : F.sz - 1;
  const int32_t yp = c.y + 1 < F.sy ? c.y + 1 : c.y;
  const int32_t ym = c.y > 0 ? c.y - 1 : c.y;
  const double vi = x[i] + cxv[parent(F, C, c.x, c.y, c.z)];
  const double kv =
      b.wxp * (vi - x[b.xp] - cxv[parent(F, C, xp, c.y, c.z)]) +
      b.wxm * (vi - x[b.xm] - cxv[parent(F, C, xm, c.y, c.z)]) +
      b.wyp * (vi - x[b.yp] - cxv[parent(F, C, c.x, yp, c.z)]) +
      b.wym * (vi - x[b.ym] - cxv[parent(F, C, c.x, ym, c.z)]) +
      b.wzp * (vi - x[b.zp] - cxv[parent(F, C, c.x, c.y, zp)]) +
      b.wzm * (vi - x[b.zm] - cxv[parent(F, C, c.x, c.y, zm)]);
  res[i] = r[i] - kv;
}

__global__ void __launch_bounds__(kBlock)
    k_mg_prolong_resid(MgLevel F, const double *__restrict__ r,
                       const double *__restrict__ x, double *__restrict__ res,
                       MgLevel C, const int *done) {
  MG_DONE_RETURN;
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F.n) return;
  prolong_resid_at(F, r, x, res, C, i);
}

// ---------------------------------------------------------------------------
// coarse levels

// exact solve of the singular coarsest line problem, projected to zero mean;
// executed by a whole CTA
__device__ __forceinline__ void coarsest_block(const MgLevel &L) {
  if (threadIdx.x == 0) line_solve<0>(L, 0, 0, L.r, L.x, L.x, 1.0);
  __syncthreads();
  double v[1] = {0.0};
  for (int32_t i = threadIdx.x; i < L.n; i += blockDim.x) v[0] += L.x[i];
  block_reduce<1>(v);
  __shared__ double mean;
  if (threadIdx.x == 0) mean = v[0] / (double)L.n;
  __syncthreads();
  for (int32_t i = threadIdx.x; i < L.n; i += blockDim.x) L.x[i] -= mean;
}

__global__ void __launch_bounds__(kBlock)
    k_mg_coarsest(MgLevel L, const int *done) {
  MG_DONE_RETURN;
  coarsest_block(L);
}

// The V-cycle from level l0 down in ONE CTA: the small coarse levels are
// latency-bound, so phases are separated by __syncthreads instead of kernel
// boundaries.  A non-singular coarsest level (coarsening stopped on odd
// sizes) gets 5 damped line sweeps.
__global__ void __launch_bounds__(1024)
    k_mg_coarse_fused(MgHierarchy h, int l0, const int *done) {
  MG_DONE_RETURN;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int last = h.nlev - 1;
  const double om = h.omega;
  for (int l = l0; l < last; ++l) {
    const MgLevel &L = h.lv[l], &C = h.lv[l + 1];
    for (int32_t ln = tid; ln < L.sx * L.sz; ln += nt)
      line_solve<0>(L, ln / L.sz, ln % L.sz, L.r, L.x, L.x, om);
    __syncthreads();
    for (int32_t I = tid; I < C.n; I += nt)
      resid_restrict_at(L, L.r, L.x, C, I, h.corr);
    __syncthreads();
  }
  const MgLevel &E = h.lv[last];
  if (E.pinned) {
    coarsest_block(E);
  } else {
    for (int32_t ln = tid; ln < E.sx * E.sz; ln += nt)
      line_solve<0>(E, ln / E.sz, ln % E.sz, E.r, E.x, E.x, om);
    __syncthreads();
    for (int it = 0; it < 4; ++it) {
      for (int32_t i = tid; i < E.n; i += nt)
        E.t[i] = E.r[i] - kx(nbhd(E, decode(E, i)), i, E.x);
      __syncthreads();
      for (int32_t ln = tid; ln < E.sx * E.sz; ln += nt)
        line_solve<0>(E, ln / E.sz, ln % E.sz, E.t, E.t, E.t, om);
      __syncthreads();
      for (int32_t i = tid; i < E.n; i += nt) E.x[i] += E.t[i];
      __syncthreads();
    }
  }
  __syncthreads();
  for (int l = last - 1; l >= l0; --l) {
    const MgLevel &L = h.lv[l], &C = h.lv[l + 1];
    for (int32_t i = tid; i < L.n; i += nt)
      prolong_resid_at(L, L.r, L.x, L.t, C, i);
    __syncthreads();
    for (int32_t ln = tid; ln < L.sx * L.sz; ln += nt)
      line_solve<2>(L, ln / L.sz, ln % L.sz, L.t, L.t, L.x, om, &C);
    __syncthreads();
  }
}

// The same V-cycle with every array of levels l0 .. last staged in shared
// memory (small hierarchies: C1's coarse levels are ~22 KB): the serial
// Thomas sweeps and the restrictions then chain on shared-memory latency
// instead of L2 latency.  In: the coefficient arrays and level l0's rhs;
// out: level l0's solution.  The level descriptors live in shared memory
// too, their array pointers redirected to the staged copies.  From l0 = 0
// (a whole small hierarchy: C1's 1,024-cell cavity) it is the entire
// V-cycle in one launch instead of five, and with `fz.st` its last
// smoothing sweep also forms the CG z-sums and beta (k_mg_smooth2_cg's
// fusion, reduced over the block).
constexpr int kStagedThreads = 256;  // 255 registers: line_solve's chunks
                                     // stay in registers (512: spills)
__global__ void __launch_bounds__(kStagedThreads)
    k_mg_coarse_staged(MgHierarchy h, int l0, CgFuse fz, const int *done) {
  MG_DONE_RETURN;
  extern __shared__ __align__(16) double shm[];
  __shared__ MgLevel slv[kMgMaxLevels];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int last = h.nlev - 1;
  const double om = h.omega;
  if (tid == 0) {
    double *p = shm;
    for (int l = l0; l <= last; ++l) {
      MgLevel L = h.lv[l];
      double **arr[8] = {&L.wx, &L.wy, &L.wz, &L.cp, &L.ivd,
                         &L.r, &L.x, &L.t};
      for (int k = 0; k < 8; ++k)
        if (*arr[k]) {
          *arr[k] = p;
          p += L.n;
        }
      slv[l] = L;
    }
  }
  __syncthreads();
  for (int l = l0; l <= last; ++l) {
    const MgLevel &G = h.lv[l], &S = slv[l];
    const double *src[6] = {G.wx, G.wy, G.wz, G.cp, G.ivd,
                            l == l0 ? G.r : nullptr};
    double *dst[6] = {S.wx, S.wy, S.wz, S.cp, S.ivd, S.r};
    for (int k = 0; k < 6; ++k)
      if (src[k])
        for (int32_t i = tid; i < G.n; i += nt) dst[k][i] = src[k][i];
  }
  __syncthreads();
  for (int l = l0; l < last; ++l) {
    const MgLevel &L = slv[l], &C = slv[l + 1];
    for (int32_t ln = tid; ln < L.sx * L.sz; ln += nt)
      line_solve<0>(L, ln / L.sz, ln % L.sz, L.r, L.x, L.x, om);
    __syncthreads();
    for (int32_t I = tid; I < C.n; I += nt)
      resid_restrict_at(L, L.r, L.x, C, I, h.corr);
    __syncthreads();
  }
  const MgLevel &E = slv[last];
  if (E.pinned) {
    coarsest_block(E);
  } else {
    for (int32_t ln = tid; ln < E.sx * E.sz; ln += nt)
      line_solve<0>(E, ln / E.sz, ln % E.sz, E.r, E.x, E.x, om);
    __syncthreads();
    for (int it = 0; it < 4; ++it) {
      for (int32_t i = tid; i < E.n; i += nt)
        E.t[i] = E.r[i] - kx(nbhd(E, decode(E, i)), i, E.x);
      __syncthreads();
      for (int32_t ln = tid; ln < E.sx * E.sz; ln += nt)
        line_solve<0>(E, ln / E.sz, ln % E.sz, E.t, E.t, E.t, om);
      __syncthreads();
      for (int32_t i = tid; i < E.n; i += nt) E.x[i] += E.t[i];
      __syncthreads();
    }
  }
  __syncthreads();
  const bool sums_on = l0 == 0 && fz.st;
  double sums[3] = {0.0, 0.0, 0.0};
  for (int l = last - 1; l >= l0; --l) {
    const MgLevel &L = slv[l], &C = slv[l + 1];
    for (int32_t i = tid; i < L.n; i += nt)
      prolong_resid_at(L, L.r, L.x, L.t, C, i);
    __syncthreads();
    for (int32_t ln = tid; ln < L.sx * L.sz; ln += nt) {
      if (l == 0 && sums_on)
        line_solve<2, true>(L, ln / L.sz, ln % L.sz, L.t, L.t, L.x, om, &C,
                            sums);
      else
        line_solve<2>(L, ln / L.sz, ln % L.sz, L.t, L.t, L.x, om, &C);
    }
    __syncthreads();
  }
  if (sums_on) {
    block_reduce<3>(sums);
    if (tid == 0)
      cg_fin_z(fz.st, sums[0], sums[1], sums[2], (int32_t)slv[0].n,
               fz.initial != 0);
  }
  const double *xs = slv[l0].x;
  double *xg = h.lv[l0].x;
  for (int32_t i = tid; i < h.lv[l0].n; i += nt) xg[i] = xs[i];
}

// shared-memory bytes k_mg_coarse_staged needs for levels l0 .. last
static size_t coarse_staged_bytes(const MgHierarchy &h, int l0) {
  size_t b = 0;
  for (int l = l0; l < h.nlev; ++l) {
    const MgLevel &L = h.lv[l];
    const double *arr[8] = {L.wx, L.wy, L.wz, L.cp, L.ivd, L.r, L.x, L.t};
    for (int k = 0; k < 8; ++k)
      if (arr[k]) b += sizeof(double) * (size_t)L.n;
  }
  return b;
}
constexpr size_t kCoarseStagedMax = 160 * 1024;

static bool staged_ok(const MgHierarchy &h, int l0) {
  return coarse_staged_bytes(h, l0) <= kCoarseStagedMax &&
         !getenv("PF_MG_NO_STAGE");
}

static void launch_coarse(const MgHierarchy &h, int l0, cudaStream_t s,
                          const int *done,
                          CgFuse fz = CgFuse{nullptr, nullptr, nullptr, 0}) {
  const size_t b = coarse_staged_bytes(h, l0);
  if (!staged_ok(h, l0)) {
    launch(k_mg_coarse_fused, 1, 1024, s, h, l0, done);
    return;
  }
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_mg_coarse_staged,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kCoarseStagedMax);
  });
  count_launch();
  k_mg_coarse_staged<<<1, kStagedThreads, b, s>>>(h, l0, fz, done);
}

// CG z-sums for the rare single-level hierarchy (no final smoother to fuse)
__global__ void __launch_bounds__(kBlock)
    k_mg_zsum(const double *__restrict__ r, const double *__restrict__ z,
              int32_t n, CgFuse fz, const int *done) {
  MG_DONE_RETURN;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    acc[0] += z[i];
    acc[1] += r[i] * z[i];
    acc[2] += r[i];
  }
  double tot[3];
  if (grid_reduce<3>(acc, fz.partials, fz.counter, tot))
    cg_fin_z(fz.st, tot[0], tot[1], tot[2], n, fz.initial != 0);
}

// ---------------------------------------------------------------------------
// host side

// level-0 face weights of the spectral mode, padded for the arrays after it
static int64_t spec_level0_bytes(int64_t n) {
  return (3 * n * 8 + 255) / 256 * 256;
}

bool mg_plan(const Plan &p, MgHierarchy &h, int64_t *bytes) {
  h.nlev = 0;
  h.omega = 0.85;
  h.corr = 1.0;
  if (const char *e = getenv("PF_MG_CORR")) h.corr = atof(e);
  h.spectral = 0;
  *bytes = 0;
  if (p.d.topo != PF_TOPO_BOX) return false;
  const int d = p.d.dim;
  int sx, sy, sz, px, pz;
  if (d == 3) {
    h.ax_of[0] = 0;
    h.ax_of[1] = 1;
    h.ax_of[2] = 2;
    sx = (int)p.d.box_shape[0];
    sy = (int)p.d.box_shape[1];
    sz = (int)p.d.box_shape[2];
    px = p.d.box_periodic[0];
    pz = p.d.box_periodic[2];
    if (p.d.box_periodic[1]) return false;
  } else {
    h.ax_of[0] = -1;
    h.ax_of[1] = 0;
    h.ax_of[2] = 1;
    sx = 1;
    sy = (int)p.d.box_shape[0];
    sz = (int)p.d.box_shape[1];
    px = 0;
    pz = p.d.box_periodic[1];
    if (p.d.box_periodic[0]) return false;
  }
  if (sy < 2 || (sx <= 1 && sz <= 1)) return false;
  h.spectral = 0;
  // slab plans: the spectral solve transforms the global X axis (all-to-all
  // over the ranks); the coarse levels of the multigrid are not distributed
  const int sxg = p.slab ? (int)p.d.slab_nx : sx;
  if (p.slab && (d != 3 || p.d.geom_precond != PF_GEOM_SPECTRAL ||
                 !spec_ok(d, sxg, sy, sz, px, pz) || (p.nxl * sy) % 2))
    return false;
  if (p.d.geom_precond == PF_GEOM_SPECTRAL && spec_ok(d, sxg, sy, sz, px, pz)) {
    // level 0 face weights + the spectral solve, no coarse levels
    MgLevel &L = h.lv[0];
    L = MgLevel{};
    L.sx = sx;
    L.sy = sy;
    L.sz = sz;
    L.px = px;
    L.pz = pz;
    L.n = (int64_t)sx * sy * sz;
    L.fx = L.fy = L.fz = 1;
    h.nlev = 1;
    h.spectral = 1;
    spec_plan(h.sp, sxg, sy, sz);
    if (p.slab)
      spec_slab_plan(h.sp, (int)p.nxl, (int)p.d.slab_x0, p.d.slab_rank,
                     p.d.slab_world);
    *bytes = spec_level0_bytes(L.n) + spec_bytes(h.sp);
    return true;
  }
  int64_t total = 0;
  for (;;) {
    MgLevel &L = h.lv[h.nlev];
    L = MgLevel{};
    L.sx = sx;
    L.sy = sy;
    L.sz = sz;
    L.px = px;
    L.pz = pz;
    L.n = (int64_t)sx * sy * sz;
    L.fx = (sx % 2 == 0) ? 2 : 1;
    L.fy = (sy % 2 == 0 && sy > 2) ? 2 : 1;
    L.fz = (sz % 2 == 0) ? 2 : 1;
    total += (h.nlev == 0 ? 6 : 8) * L.n;
    ++h.nlev;
    const bool last = (L.fx == 1 && L.fz == 1) || h.nlev == kMgMaxLevels;
    if (last) {
      L.fx = L.fy = L.fz = 1;
      L.pinned = (sx == 1 && sz == 1);
      break;
    }
    sx /= L.fx;
    sy /= L.fy;
    sz /= L.fz;
  }
  *bytes = total * 8;
  return true;
}

void mg_bind(MgHierarchy &h, void *base) {
  double *q = static_cast<double *>(base);
  if (h.spectral) {
    MgLevel &L = h.lv[0];
    L.wx = q;
    L.wy = q + L.n;
    L.wz = q + 2 * L.n;
    L.cp = L.ivd = L.t = L.r = L.x = nullptr;
    spec_bind(h.sp, static_cast<char *>(base) + spec_level0_bytes(L.n));
    return;
  }
  for (int k = 0; k < h.nlev; ++k) {
    MgLevel &L = h.lv[k];
    L.wx = q;
    q += L.n;
    L.wy = q;
    q += L.n;
    L.wz = q;
    q += L.n;
    L.cp = q;
    q += L.n;
    L.ivd = q;
    q += L.n;
    L.t = q;
    q += L.n;
    if (k > 0) {
      L.r = q;
      q += L.n;
      L.x = q;
      q += L.n;
    } else {
      L.r = L.x = nullptr;
    }
  }
}

static int lines_grid(const MgLevel &L) {
  return grid_for((int64_t)L.sx * L.sz, kLineBlock);
}

int mg_setup(const MgHierarchy &h, const double *k, int64_t n, cudaStream_t s,
             const int *done, const Plan *pl) {
  launch(k_mg_faces0, grid_for(n), kBlock, s, h.lv[0], k, n, h.ax_of[0],
         h.ax_of[1], h.ax_of[2], done);
  if (h.spectral) return spec_setup(h.lv[0], h.sp, s, done, pl);
  for (int l = 0; l + 1 < h.nlev; ++l)
    launch(k_mg_aggregate, grid_for(h.lv[l + 1].n), kBlock, s, h.lv[l],
           h.lv[l + 1], done);
  for (int l = 0; l < h.nlev; ++l)
    launch(k_mg_factor, grid_for((int64_t)h.lv[l].sx * h.lv[l].sz), kBlock,
           s, h.lv[l], done);
  PF_LAUNCH_CHECK("mg_setup");
  return PF_OK;
}

// cells: levels at most this small run the rest of the V-cycle in one CTA
// (a 24576-cell level is already too big for one SM; the 3072-cell and
// smaller levels are pure launch/latency cost -- measured on C4)
constexpr int64_t kFusedCoarseMax = 4096;

static void vcycle(const MgHierarchy &h, int l, const double *r, double *x,
                   cudaStream_t s, const int *done, cudaEvent_t *ev,
                   const CgFuse *fuse, int red_blocks, int fused_from) {
  auto mark = [&](int k) {
    if (ev && l == 0) cudaEventRecord(ev[k], s);
  };
  const MgLevel &L = h.lv[l];
  if (l > 0 && (l >= fused_from || (l == h.nlev - 1 && !L.pinned))) {
    launch_coarse(h, l, s, done);
    return;
  }
  if (l == h.nlev - 1) {
    launch(k_mg_coarsest, 1, kBlock, s, L, done);
    return;
  }
  const MgLevel &C = h.lv[l + 1];
  mark(0);
  launch(k_mg_smooth0, lines_grid(L), kLineBlock, s, L, r, x, h.omega, done);
  mark(1);
  launch(k_mg_resid_restrict, grid_for(C.n), kBlock, s, L, r,
         (const double *)x, C, h.corr, done);
  mark(2);
  vcycle(h, l + 1, C.r, C.x, s, done, nullptr, nullptr, red_blocks,
         fused_from);
  mark(3);
  launch(k_mg_prolong_resid, grid_for(L.n), kBlock, s, L, r,
         (const double *)x, L.t, C, done);
  mark(4);
  if (l == 0 && fuse && fuse->st)
    launch(k_mg_smooth2_cg, std::min(lines_grid(L), red_blocks), kLineBlock,
           s, L, L.t, x, h.omega, C, *fuse, done);
  else
    launch(k_mg_smooth2, lines_grid(L), kLineBlock, s, L, L.t, x, h.omega, C,
           done);
  mark(5);
}

int mg_apply(const MgHierarchy &h, const double *r, double *z, cudaStream_t s,
             const int *done, cudaEvent_t *ev, const CgFuse *fuse,
             int red_blocks, const Plan *pl) {
  MgHierarchy hh = h;
  hh.lv[0].r = const_cast<double *>(r);
  hh.lv[0].x = z;
  if (hh.spectral)
    return spec_apply(hh.lv[0], hh.sp, r, z, s, done, ev, fuse, red_blocks,
                      pl);
  int fused_from = hh.nlev;
  for (int l = 1; l < hh.nlev; ++l)
    if (hh.lv[l].n <= kFusedCoarseMax) {
      fused_from = l;
      break;
    }
  if (hh.nlev == 1) {
    // the whole problem is one level: exact (pinned) or fused sweeps
    if (hh.lv[0].pinned)
      launch(k_mg_coarsest, 1, kBlock, s, hh.lv[0], done);
    else
      launch(k_mg_coarse_fused, 1, 1024, s, hh, 0, done);
    if (fuse && fuse->st)
      launch(k_mg_zsum, std::min(grid_for(hh.lv[0].n), red_blocks), kBlock,
             s, (const double *)r, (const double *)z, (int32_t)hh.lv[0].n,
             *fuse, done);
  } else if (!ev && hh.lv[0].n <= kFusedCoarseMax && staged_ok(hh, 0) &&
             (!fuse || fuse->st)) {
    // a whole small hierarchy: one staged single-CTA V-cycle (the level-0
    // passes are latency, not bandwidth, at a few thousand cells)
    launch_coarse(hh, 0, s, done,
                  fuse ? *fuse : CgFuse{nullptr, nullptr, nullptr, 0});
  } else {
    vcycle(hh, 0, r, z, s, done, ev, fuse, red_blocks, fused_from);
  }
  PF_LAUNCH_CHECK("mg_apply");
  return PF_OK;
}

}  // namespace pf
