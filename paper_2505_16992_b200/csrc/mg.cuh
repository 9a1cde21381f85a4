// mg.cuh -- geometric multigrid preconditioner for the pressure operator on
// single-block (box) grids.
//
// Replaces the reference's ILU(0) preconditioner (S/linalg.py:88-108,
// S/_kernels_c.pyx:66-149), whose triangular solves are sequential, with a
// symmetric V(1,1)-cycle that is a fixed SPD operator on the zero-mean
// subspace, so CG keeps its guarantees and converges to the same discrete
// solution (only iteration counts change):
//
//  * canonical axes (X, Y, Z): Y is the LINE axis (the wall-normal, refined
//    axis of the channel / the first axis in 2D);
//  * smoother: damped (omega = 0.85) block-Jacobi with exact tridiagonal
//    solves along the Y lines (one thread per line, coalesced across lines),
//    which removes the wall-refinement anisotropy;
//  * coarsening: 2 along X, Y, Z while the axis is even (Y while longer than
//    2); coarse operators are Galerkin with piecewise-constant aggregation,
//    i.e. coarse face weights are sums of fine face weights, so every level
//    keeps the symmetric 7-point face form with exact zero row sums;
//  * coarsest level (X = Z = 1): the singular Y-line Neumann problem, solved
//    exactly by a pinned Thomas sweep and projected to zero mean; levels of
//    at most a few thousand cells run as one CTA (latency, not bandwidth).
//
// Measured alternative (not used): a red-black line Gauss-Seidel smoother
// cut iterations by ~22 % on the C4 channel but doubled the time per
// iteration, because each colour pass has only half of the lines in flight
// for the serial Thomas recurrences.
#pragma once

#include "cgstate.cuh"
#include "common.cuh"

namespace pf {

// ---- level stencil helpers (shared with the CG kernels) ----

struct Cell3 {
  int32_t x, y, z, i;
};

__device__ __forceinline__ Cell3 decode(const MgLevel &L, int32_t i) {
  Cell3 c;
  c.i = i;
  c.z = i % L.sz;
  const int32_t t = i / L.sz;
  c.y = t % L.sy;
  c.x = t / L.sy;
  return c;
}

// the six faces of a cell: neighbour indices and weights (X/Z periodic or
// walled, Y walled)
struct Nbhd {
  int32_t xp, xm, yp, ym, zp, zm;
  double wxp, wxm, wyp, wym, wzp, wzm;
};

__device__ __forceinline__ Nbhd nbhd(const MgLevel &L, const Cell3 &c) {
  Nbhd b;
  const int32_t sX = L.sy * L.sz, sY = L.sz;
  b.xp = c.x + 1 < L.sx ? c.i + sX : c.i - (L.sx - 1) * sX;
  b.xm = c.x > 0 ? c.i - sX : c.i + (L.sx - 1) * sX;
  b.zp = c.z + 1 < L.sz ? c.i + 1 : c.i - (L.sz - 1);
  b.zm = c.z > 0 ? c.i - 1 : c.i + (L.sz - 1);
  b.yp = c.y + 1 < L.sy ? c.i + sY : c.i;
  b.ym = c.y > 0 ? c.i - sY : c.i;
  b.wxp = L.wx[c.i];
  b.wxm = (c.x > 0 || L.px) ? L.wx[b.xm] : 0.0;
  b.wzp = L.wz[c.i];
  b.wzm = (c.z > 0 || L.pz) ? L.wz[b.zm] : 0.0;
  b.wyp = L.wy[c.i];
  b.wym = c.y > 0 ? L.wy[b.ym] : 0.0;
  return b;
}

__device__ __forceinline__ double kx(const Nbhd &b, int32_t i,
                                     const double *v) {
  const double vi = v[i];
  return b.wxp * (vi - v[b.xp]) + b.wxm * (vi - v[b.xm]) +
         b.wyp * (vi - v[b.yp]) + b.wym * (vi - v[b.ym]) +
         b.wzp * (vi - v[b.zp]) + b.wzm * (vi - v[b.zm]);
}

// Host: plan the hierarchy for a box plan; returns false when MG does not
// apply (gather topology, periodic line axis, line axis shorter than 2).
bool mg_plan(const Plan &p, MgHierarchy &h, int64_t *bytes);
// Host: carve level arrays out of a device buffer of the planned size.
void mg_bind(MgHierarchy &h, void *base);
// Setup for operator K (2d+1 stencil, K = -P): level-0 faces, coarse
// aggregation, line factorisations.
int mg_setup(const MgHierarchy &h, const double *k_stencil, int64_t n,
             cudaStream_t s, const int *all_done, const Plan *pl = nullptr);
// z = V(r) on the fine level; every kernel returns at once when *all_done.
// `ev` (optional, 6 events) is recorded around the level-0 kernels:
// smooth | restrict | coarse levels | prolong | smooth.  `fuse` (optional)
// folds the CG z-sums and beta into the final level-0 smoothing pass (no
// separate z-sum kernel); it needs red_blocks.
int mg_apply(const MgHierarchy &h, const double *r, double *z,
             cudaStream_t s, const int *all_done, cudaEvent_t *ev = nullptr,
             const CgFuse *fuse = nullptr, int red_blocks = 0,
             const Plan *pl = nullptr);

}  // namespace pf
