// common.cuh -- plan view, mesh topologies, deterministic reductions.
//
// Everything here is device-side plumbing shared by the forward, solver and
// adjoint translation units.  The cell-adjacency semantics follow the
// reference mesh (S/mesh.py:294-321): for cell i and face f = 2a + s the
// neighbour is nbr[a, s, i] (or a boundary face), the neighbour's axis seen
// across the face is nbr_ax[a, s, i, a] and its orientation nbr_sign.
#pragma once

#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <initializer_list>
#include <string>

#include "../../include/pisob200.h"
#include "comm.cuh"

namespace pf {

constexpr int kBlock = 256;      // threads per CTA for streaming kernels
constexpr int kMaxRedBlocks = 1184;  // 148 SMs x 8 resident CTAs
constexpr int kMaxK = 12;        // values per fused reduction

void set_error(const std::string &msg);
int cuda_check(cudaError_t e, const char *what);
#define PF_CUDA(call)                                          \
  do {                                                         \
    int _rc = ::pf::cuda_check((call), #call);                 \
    if (_rc) return _rc;                                       \
  } while (0)
#define PF_LAUNCH_CHECK(what) PF_CUDA(cudaGetLastError())

// Every kernel launch of the library goes through launch(), which counts it
// (pf_launch_count) -- the bench reports how many of OUR kernels ran.
// Atomic: the in-process slab tests drive several plans from concurrent host
// threads.  Graph capture counts its kernels in a thread-local counter
// (g_capture_count) instead of rewinding the global one.
extern std::atomic<unsigned long long> g_launches;
extern thread_local unsigned long long *g_capture_count;
inline void count_launch() {
  if (g_capture_count)
    ++*g_capture_count;
  else
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                   cudaStream_t stream, Args... args) {
  count_launch();
  kernel<<<grid, block, 0, stream>>>(args...);
}

// Multigrid hierarchy of a box plan (see mg.cuh); arrays are bound to the
// caller's MG workspace on every call.
constexpr int kMgMaxLevels = 16;

struct MgLevel {
  int32_t sx, sy, sz;   // canonical dims
  int32_t px, pz;       // periodic X / Z
  int32_t fx, fy, fz;   // coarsening factors to the next level
  int32_t pinned;       // singular coarsest line problem
  int64_t n;
  double *wx, *wy, *wz;  // +face weights
  double *cp, *ivd;      // Thomas factors along Y
  double *r, *x, *t;     // level rhs, solution, scratch
};

// Spectral preconditioner of a box with periodic, uniformly spaced X and Z
// (see spectral.cuh): exact inverse of the XZ-plane-averaged operator.
struct SpecPlan {
  int32_t sx, sy, sz;  // canonical dims (sx == 1 in 2D); sx is GLOBAL
  int32_t nkz;         // sz / 2 + 1 retained Z wavenumbers
  int32_t lpx, lpz;    // lines per CTA of the X / Z transforms
  // slab decomposition of X (comm.cuh): this rank owns X lines
  // x0 .. x0 + nxl - 1 (stored at local plane x + xoff) and the Z
  // wavenumbers kz0[rank] .. kz0[rank + 1] - 1 of the transposed spectrum;
  // peer_s[q] is rank q's work array (own at [rank]).  Single GPU: nxl = sx,
  // xoff = x0 = 0, one rank owning every kz.
  int32_t nxl, xoff, x0, rank, world;
  int32_t kz0[kMaxRanks + 1];
  double2 *peer_s[kMaxRanks];
  double2 *s;          // (sy, kz of this rank, sx) spectral work array
  double *cw;          // (sy, nkz * sx) Thomas c'
  double *iw;          // (sy, nkz * sx) Thomas 1 / den
  double *ax, *ay, *az;  // (sy) plane-mean face weights
  double2 *twx, *twz;    // exp(-2 pi i k / N), N = sx, sz
  double *lx, *lz;       // 2 - 2 cos(2 pi k / N)
};

struct MgHierarchy {
  int nlev;
  int ax_of[3];  // physical axis of canonical X, Y, Z (-1: absent)
  MgLevel lv[kMgMaxLevels];
  double omega;   // damping of the block-Jacobi line smoother
  double corr;    // coarse-correction scale (restricted residual x corr)
  int spectral;   // level 0 only, preconditioned by the spectral solve
  SpecPlan sp;
};


// Cached CUDA graph of the multigrid CG iteration (keyed by the buffers it
// was captured on) and the private stream used for capturing it.
struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  const void *key[3] = {nullptr, nullptr, nullptr};
  unsigned long long nkern = 0;
};

struct CommHost;

// Host-side plan: the immutable device description plus derived launch
// parameters.
struct Plan {
  pf_plan_desc d;
  int num_sms;
  int red_blocks;  // grid of reduction kernels
  bool has_mg;     // geometric multigrid available for this topology
  MgHierarchy mg;
  int64_t mg_bytes;
  mutable GraphCache graph;
  // slab decomposition along axis 0 (comm.cuh): owned cells [i0, i1) of the
  // (nxl + 2)-plane local box; i0 = 0, i1 = n otherwise
  bool slab = false;
  int32_t i0 = 0, i1 = 0;
  double ng = 0.0;  // owned cells summed over all ranks
  int64_t plane = 0, nxl = 0;
  CommHost *comm = nullptr;  // attached communicator (slab plans)
  // pinned staging for the small device-to-host reads (solver state,
  // scalars): a copy into pageable memory is staged through a buffer the
  // driver shares between streams, which would serialise slabs that share
  // a device
  void *pinned = nullptr;
  void *pinned_dev = nullptr;  // its device alias (mapped)
  // lock-step iterations of the last BiCGStab solve (plain, transposed):
  // the first batch the next solve launches before polling
  mutable int bi_hint[2] = {0, 0};
};

constexpr size_t kPinnedBytes = 4096;
// copy `bytes` (<= kPinnedBytes) from device to host through the plan's
// pinned buffer and wait for it (stream ordered)
int d2h(const Plan &p, void *host, const void *dev, size_t bytes,
        cudaStream_t s);

// owned cell range of a plan, for the pointwise kernels
struct Rng {
  int32_t i0, i1;
  double ng;
};
inline Rng plan_range(const Plan &p) { return Rng{p.i0, p.i1, p.ng}; }
#define RANGE_LOOP(i, rg)                                                  \
  for (int32_t i = (rg).i0 + blockIdx.x * blockDim.x + threadIdx.x;        \
       i < (rg).i1; i += gridDim.x * blockDim.x)

// halo exchange of the ghost planes of a set of arrays (no-op unless the
// plan is a slab plan with a communicator), barrier, vector allreduce
int halo_exchange(const Plan &p, const HaloItem *items, int count,
                  cudaStream_t s);
inline int halo(const Plan &p, cudaStream_t s,
                std::initializer_list<HaloItem> items) {
  return halo_exchange(p, items.begin(), (int)items.size(), s);
}
int comm_barrier(const Plan &p, cudaStream_t s);
// PF_ERR_CUDA (with the details) once a device-side peer wait timed out
int comm_check(const Plan &p, cudaStream_t s);
int comm_vec_allreduce(const Plan &p, double *buf, int k, int op,
                       cudaStream_t s);
// any length (chunks of the vector slot)
int comm_vec_allreduce_n(const Plan &p, double *buf, int64_t k, int op,
                         cudaStream_t s);

// ---------------------------------------------------------------------------
// face lookup

struct Face {
  int32_t nb;    // neighbour cell, -1 for a boundary face
  int32_t ax;    // neighbour's axis for my face axis (perm[a])
  int32_t neg;   // orientation flip of that axis (sign == -1)
  int32_t bidx;  // boundary entry when nb < 0
};

// back face of the neighbour pointing at me: axis perm[a], side flipped
// unless the orientation is reversed (S/mesh.py:393-397)
__device__ __forceinline__ int back_face(const Face &fc, int s) {
  const int rs = fc.neg ? s : 1 - s;
  return 2 * fc.ax + rs;
}

struct GatherTopo {
  static constexpr bool kBox = false;
  const int32_t *nbr;
  int64_t n;
  struct Cell {
    int32_t i;
  };
  __device__ __forceinline__ Cell cell(int32_t i) const { return Cell{i}; }
  __device__ __forceinline__ Face face(const Cell &c, int f) const {
    const int32_t v = __ldg(nbr + (int64_t)f * n + c.i);
    Face r;
    if (v >= 0) {
      r.nb = v & 0x03FFFFFF;
      r.ax = (v >> 26) & 3;
      r.neg = (v >> 28) & 1;
      r.bidx = -1;
    } else {
      r.nb = -1;
      r.ax = f >> 1;
      r.neg = 0;
      r.bidx = ~v;
    }
    return r;
  }
};

// quotient of a non-negative int32 by a positive divisor through a double
// reciprocal (exact after the +-1 correction; cheaper than the ~20
// instruction integer division with a runtime divisor)
__device__ __forceinline__ int32_t fast_div(int32_t i, int32_t d,
                                            double inv) {
  int32_t q = __double2int_rz((double)i * inv);
  int32_t r = i - q * d;
  if (r < 0) --q;
  else if (r >= d) ++q;
  return q;
}

template <int D>
struct BoxTopo {
  static constexpr bool kBox = true;
  int32_t shape[3];
  int32_t stride[3];
  int32_t periodic[3];
  int32_t face_off[6];
  double inv_stride[3];  // 1 / stride (fast_div)
  double inv_shape[3];   // 1 / shape
  struct Cell {
    int32_t i;
    int32_t x[3];
  };
  __device__ __forceinline__ Cell cell(int32_t i) const {
    Cell c;
    c.i = i;
    int32_t rem = i;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      c.x[a] = a == D - 1 ? rem : fast_div(rem, stride[a], inv_stride[a]);
      rem -= c.x[a] * stride[a];
    }
    return c;
  }
  __device__ __forceinline__ Face face(const Cell &c, int f) const {
    const int a = f >> 1, s = f & 1;
    Face r;
    r.ax = a;
    r.neg = 0;
    r.bidx = -1;
    const int xa = c.x[a];
    if (s) {
      if (xa + 1 < shape[a]) {
        r.nb = c.i + stride[a];
      } else if (periodic[a]) {
        r.nb = c.i - (shape[a] - 1) * stride[a];
      } else {
        r.nb = -1;
      }
    } else {
      if (xa > 0) {
        r.nb = c.i - stride[a];
      } else if (periodic[a]) {
        r.nb = c.i + (shape[a] - 1) * stride[a];
      } else {
        r.nb = -1;
      }
    }
    if (r.nb < 0) {
      // boundary entries are the face's cells in C order of the other axes
      int32_t idx = 0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        if (k == a) continue;
        idx = idx * shape[k] + c.x[k];
      }
      r.bidx = face_off[f] + idx;
    }
    return r;
  }
};

// Device view of the plan (passed by value into kernels).
template <int D, class Topo>
struct View {
  static constexpr int kDim = D;
  using Cell = typename Topo::Cell;
  Topo topo;
  int32_t n;
  int32_t m;
  int32_t i0, i1;  // owned cells (the whole range unless a slab plan)
  double ng;       // owned cells over all ranks (means, zero-mean projection)
  const double *__restrict__ jac;
  const double *__restrict__ ijac;   // 1 / jac (or null)
  const double *__restrict__ tmat;   // (D*D, n)
  const double *__restrict__ alpha;  // (D, n)
  const int32_t *__restrict__ bcell;
  const int32_t *__restrict__ bface;
  const double *__restrict__ bjac;
  const double *__restrict__ bt;  // (D, m)
  const double *__restrict__ balpha;
  // non-orthogonal grids only
  const double *__restrict__ alpha_full;  // (D*D, n)
  const double *__restrict__ balpha_row;  // (D, m) face alpha[a][k]
  const int32_t *__restrict__ bfid;       // (m) face id
  const int32_t *__restrict__ finfo;      // (nfaces, 8)
  int32_t has_cross;
  // separable box metrics (sep != 0): 1-D widths and inverse widths; T
  // (9 values per cell, diagonal) is formed from them
  int32_t sep;
  const double *__restrict__ sdx[3];
  const double *__restrict__ sinv[3];

  __device__ __forceinline__ int32_t coord(int a, int32_t i) const {
    if constexpr (Topo::kBox) {
      const int32_t q = a == 0 ? i : fast_div(i, topo.stride[a],
                                              topo.inv_stride[a]);
      if (a == 0) return fast_div(i, topo.stride[0], topo.inv_stride[0]);
      return q - fast_div(q, topo.shape[a], topo.inv_shape[a]) * topo.shape[a];
    } else {
      return 0;
    }
  }

  __device__ __forceinline__ Rng rng() const { return Rng{i0, i1, ng}; }
  __host__ __device__ __forceinline__ int32_t owned() const { return i1 - i0; }
  __device__ __forceinline__ double AF(int a, int k, int32_t i) const {
    return __ldg(alpha_full + (int64_t)(a * D + k) * n + i);
  }
  __device__ __forceinline__ double T(int a, int j, int32_t i) const {
    if (Topo::kBox && sep)
      return a == j ? __ldg(sinv[a] + coord(a, i)) : 0.0;
    return __ldg(tmat + (int64_t)(a * D + j) * n + i);
  }
  // J and alpha stay full (n) arrays: their callers gather them at the
  // neighbours, where decoding coordinates would cost more than the load
  __device__ __forceinline__ double J(int32_t i) const {
    return __ldg(jac + i);
  }
  // 1.0 / J(i), bitwise (a load where the plan carries the array)
  __device__ __forceinline__ double IJ(int32_t i) const {
    return ijac ? __ldg(ijac + i) : 1.0 / __ldg(jac + i);
  }
  __device__ __forceinline__ double A(int a, int32_t i) const {
    return __ldg(alpha + (int64_t)a * n + i);
  }
  // contravariant flux component a of a (D, n) SoA velocity at cell i
  __device__ __forceinline__ double flux(const double *__restrict__ u, int a,
                                         int32_t i) const {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) acc += T(a, j, i) * u[(int64_t)j * n + i];
    return J(i) * acc;
  }
  // boundary face flux U_f = J_f T_f[a,:] . ub  (S/piso.py:128-131)
  __device__ __forceinline__ double bflux(const double *__restrict__ bc,
                                          int32_t e) const {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j)
      acc += __ldg(bt + (int64_t)j * m + e) * bc[(int64_t)j * m + e];
    return __ldg(bjac + e) * acc;
  }
};

template <int D, class Topo>
View<D, Topo> make_view(const Plan &p, const Topo &topo) {
  View<D, Topo> v;
  v.topo = topo;
  v.n = (int32_t)p.d.n;
  v.m = (int32_t)p.d.m;
  v.i0 = p.i0;
  v.i1 = p.i1;
  v.ng = p.ng;
  v.jac = p.d.jac;
  v.ijac = p.d.ijac;
  v.tmat = p.d.tmat;
  v.alpha = p.d.alpha_diag;
  v.bcell = p.d.bcell;
  v.bface = p.d.bface;
  v.bjac = p.d.bjac;
  v.bt = p.d.bt;
  v.balpha = p.d.balpha;
  v.alpha_full = p.d.alpha_full;
  v.balpha_row = p.d.balpha_row;
  v.bfid = p.d.bfid;
  v.finfo = p.d.finfo;
  v.has_cross = p.d.has_cross;
  v.sep = p.d.sep_dx[0] != nullptr && p.d.sep_inv[0] != nullptr;
  for (int a = 0; a < 3; ++a) {
    v.sdx[a] = p.d.sep_dx[a];
    v.sinv[a] = p.d.sep_inv[a];
  }
  return v;
}

// ---------------------------------------------------------------------------
// tangential-derivative viscous flux through a prescribed face
// (_boundary_cross_term, S/piso.py:375-392) and its adjoint
// (_adj_boundary_cross, S/adjoint.py:215-233).  A face is an area_shape grid
// of boundary entries in C order; face_grad is central inside and one-sided
// at the ends (S/piso.py:134-159).

struct FaceGeo {
  int32_t off, ndim, dims[2], st[2], j[2], active, axis;
};

template <class V>
__device__ __forceinline__ FaceGeo face_geo(const V &v, int32_t e) {
  FaceGeo g;
  const int32_t *fi = v.finfo + 8 * __ldg(v.bfid + e);
  g.off = fi[0];
  g.ndim = V::kDim - 1;
  g.dims[0] = fi[2];
  g.dims[1] = fi[3];
  g.active = fi[4];
  g.axis = fi[5];
  const int32_t l = e - g.off;
  if (V::kDim == 3) {
    g.j[0] = l / g.dims[1];
    g.j[1] = l % g.dims[1];
    g.st[0] = g.dims[1];
    g.st[1] = 1;
  } else {
    g.j[0] = l;
    g.j[1] = 0;
    g.st[0] = 1;
    g.st[1] = 0;
  }
  return g;
}

// k-th tangential axis (the q-th axis other than the face axis)
__device__ __forceinline__ int tang_axis(int axis, int q) {
  return q < axis ? q : q + 1;
}

// term[c] of the boundary cross flux at entry e (before the N nu / J scale)
template <class V>
__device__ __forceinline__ void bcross_term(const V &v, const FaceGeo &g,
                                            int32_t e,
                                            const double *__restrict__ bc,
                                            double (&term)[V::kDim]) {
  constexpr int D = V::kDim;
#pragma unroll
  for (int c = 0; c < D; ++c) term[c] = 0.0;
  for (int q = 0; q < g.ndim; ++q) {
    const int L = g.dims[q], j = g.j[q], st = g.st[q];
    const double fa = __ldg(v.balpha_row + (int64_t)tang_axis(g.axis, q) *
                                               v.m + e);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double *b = bc + (int64_t)c * v.m;
      double dub;
      if (L == 1)
        dub = 0.0;
      else if (j == 0)
        dub = b[e + st] - b[e];
      else if (j == L - 1)
        dub = b[e] - b[e - st];
      else
        dub = 0.5 * (b[e + st] - b[e - st]);
      term[c] += fa * dub;
    }
  }
}

template <int D>
BoxTopo<D> make_box(const Plan &p) {
  BoxTopo<D> t;
  int32_t st = 1;
  for (int a = D - 1; a >= 0; --a) {
    t.shape[a] = (int32_t)p.d.box_shape[a];
    t.stride[a] = st;
    st *= t.shape[a];
    t.periodic[a] = p.d.box_periodic[a];
  }
  for (int a = D; a < 3; ++a) {
    t.shape[a] = 1;
    t.stride[a] = 1;
    t.periodic[a] = 0;
  }
  for (int a = 0; a < 3; ++a) {
    t.inv_stride[a] = 1.0 / t.stride[a];
    t.inv_shape[a] = 1.0 / t.shape[a];
  }
  for (int f = 0; f < 6; ++f) t.face_off[f] = (int32_t)p.d.box_face_offset[f];
  return t;
}

// Calls fn(View<D, Topo>) with the plan's dimension and topology resolved at
// compile time.
template <class Fn>
int dispatch(const Plan &p, Fn &&fn) {
  if (p.d.topo == PF_TOPO_BOX) {
    if (p.d.dim == 2) return fn(make_view<2>(p, make_box<2>(p)));
    if (p.d.dim == 3) return fn(make_view<3>(p, make_box<3>(p)));
  } else {
    GatherTopo g{p.d.nbr, p.d.n};
    if (p.d.dim == 2) return fn(make_view<2>(p, g));
    if (p.d.dim == 3) return fn(make_view<3>(p, g));
  }
  set_error("unsupported plan dimension/topology");
  return PF_ERR_ARG;
}

inline int grid_for(int64_t work, int block = kBlock) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  return (int)g;
}

// ---------------------------------------------------------------------------
// deterministic reductions: warp shuffle tree -> per-warp smem -> per-block
// partials -> the last block to finish (ticket counter) folds the partials in
// fixed order and runs a finaliser.  No floating-point atomics anywhere.

template <int K>
__device__ __forceinline__ void warp_sum(double (&v)[K]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
  }
}

template <int K>
__device__ __forceinline__ void warp_max(double (&v)[K]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] = fmax(v[k], __shfl_down_sync(0xffffffffu, v[k], off));
  }
}

// Block-wide reduction; the result is valid in thread 0.
template <int K, bool kMax = false>
__device__ __forceinline__ void block_reduce(double (&v)[K]) {
  __shared__ double sm[32][K];  // up to 1024 threads
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (kMax) warp_max<K>(v); else warp_sum<K>(v);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[w][k] = v[k];
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] = lane < nw ? sm[lane][k] : (kMax ? -DBL_MAX : 0.0);
    if (kMax) warp_max<K>(v); else warp_sum<K>(v);
  }
  __syncthreads();
}

// Reduce K values over the whole grid; thread 0 of the last block gets the
// totals in `tot` and returns true.  partials: gridDim.x * K doubles,
// counter: one zero-initialised unsigned (reset here for the next use).
template <int K, bool kMax = false>
__device__ __forceinline__ bool grid_reduce(double (&v)[K], double *partials,
                                            unsigned *counter,
                                            double (&tot)[K]) {
  __shared__ bool is_last;
  block_reduce<K, kMax>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partials[(int64_t)blockIdx.x * K + k] = v[k];
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = kMax ? -DBL_MAX : 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double x = __ldcg(partials + (int64_t)b * K + k);
      acc[k] = kMax ? fmax(acc[k], x) : acc[k] + x;
    }
  }
  block_reduce<K, kMax>(acc);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = acc[k];
    *counter = 0u;
    // slab plans: fold the other ranks' totals in (rank order, all ranks
    // get the same bits)
    CommDev *c = ws_comm(counter);
    if (c) comm_allreduce<K, kMax>(c, tot);
    return true;
  }
  return false;
}

// Workspace layout shared by all entry points (bytes, 256-aligned):
//   [0, 4096)                 : counters (unsigned, 64), the plan's
//                               CommDev* at byte 256 (kWsCommOffset),
//                               small scalar block from byte 512
//   partials                  : kMaxRedBlocks * kMaxK doubles
//   solver scalars            : 4096 doubles
//   solver vectors            : nvec * (3 * n) doubles
struct Workspace {
  unsigned *counters;   // 64 counters
  double *scalars;      // 448 doubles of small scratch (host-visible copies)
  double *partials;     // kMaxRedBlocks * kMaxK
  double *solver;       // 4096 doubles for solver state
  double *vecs;         // vector scratch
  int64_t vec_len;      // doubles available in vecs
};
constexpr int64_t kWsHeader = 4096;
constexpr int64_t kWsSolver = 4096;
constexpr int kWsVectors = 12;  // vectors of length d*n the solvers may use

inline Workspace carve(void *base, int64_t n, int dim) {
  char *b = static_cast<char *>(base);
  Workspace w;
  w.counters = reinterpret_cast<unsigned *>(b);
  w.scalars = reinterpret_cast<double *>(b + 512);
  w.partials = reinterpret_cast<double *>(b + kWsHeader);
  w.solver = w.partials + (int64_t)kMaxRedBlocks * kMaxK;
  w.vecs = w.solver + kWsSolver;
  w.vec_len = (int64_t)kWsVectors * dim * n;
  return w;
}
inline int64_t workspace_bytes(int64_t n, int dim) {
  return kWsHeader + 8 * ((int64_t)kMaxRedBlocks * kMaxK + kWsSolver +
                          (int64_t)kWsVectors * dim * n);
}

}  // namespace pf
