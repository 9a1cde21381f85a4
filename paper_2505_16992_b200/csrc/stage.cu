// stage.cu -- the reference's wide-gradient building block and its adjoint
// as standalone device ops (S/piso.py:172-264), for the public stage API
// (paper_2505_16992_b200.piso.wide_grad / wide_grad_adjoint).  The PISO step
// itself uses the fused forms (correct_velocity, the cross fluxes); these
// entry points expose the three variants on their own, on any topology.
//
//   mirror    missing neighbour -> the cell's own value, weight 1/2
//   onesided  missing neighbour -> the cell's own value, weight 1 unless
//             both neighbours exist
//   face      missing neighbour -> a prescribed per-cell face value
//             (bc_cells), weight 1/1.5 unless both neighbours exist
//
// The adjoint is a gather: cell j collects, over each of its faces f with
// neighbour i, the contribution i's wide gradient sends along i's back face
// (np.add.at scatter of S/piso.py:261-264 restated without atomics).
#include "common.cuh"

namespace pf {

namespace {

constexpr int kMirror = 0, kOnesided = 1, kFaceVar = 2;

template <class V>
__device__ __forceinline__ double wg_weight(int variant, bool both) {
  if (variant == kMirror) return 0.5;
  if (variant == kOnesided) return both ? 0.5 : 1.0;
  return both ? 0.5 : 1.0 / 1.5;
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_wide_grad(V v, const double *__restrict__ phi, int variant,
                const double *__restrict__ bc_cells, double *__restrict__ out) {
  constexpr int D = V::kDim;
  const int32_t i = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(i);
  const double pi = phi[i];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const Face lo = v.topo.face(cell, 2 * a), hi = v.topo.face(cell, 2 * a + 1);
    double vhi, vlo;
    if (variant == kFaceVar) {
      vhi = hi.nb >= 0 ? phi[hi.nb] : bc_cells[(2 * a + 1) * n + i];
      vlo = lo.nb >= 0 ? phi[lo.nb] : bc_cells[(2 * a) * n + i];
    } else {
      vhi = hi.nb >= 0 ? phi[hi.nb] : pi;
      vlo = lo.nb >= 0 ? phi[lo.nb] : pi;
    }
    const double w = wg_weight<V>(variant, hi.nb >= 0 && lo.nb >= 0);
    out[a * n + i] = w * (vhi - vlo);
  }
}

template <class V>
__global__ void __launch_bounds__(kBlock)
    k_wide_grad_adjoint(V v, const double *__restrict__ cot, int variant,
                        double *__restrict__ out,
                        double *__restrict__ bc_cot) {
  constexpr int D = V::kDim;
  const int32_t j = v.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.i1) return;
  const int64_t n = v.n;
  const auto cell = v.topo.cell(j);
  double acc = 0.0;
#pragma unroll
  for (int f = 0; f < 2 * D; ++f) {
    const Face fc = v.topo.face(cell, f);
    if (fc.nb < 0) continue;
    // i = fc.nb reaches j through its face bf = 2 a' + s'
    const int bf = back_face(fc, f & 1);
    const int ap = bf >> 1, sp = bf & 1;
    const auto ci = v.topo.cell(fc.nb);
    const bool both = v.topo.face(ci, 2 * ap).nb >= 0 &&
                      v.topo.face(ci, 2 * ap + 1).nb >= 0;
    const double c = wg_weight<V>(variant, both) * cot[ap * n + fc.nb];
    acc += sp ? c : -c;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const Face lo = v.topo.face(cell, 2 * a), hi = v.topo.face(cell, 2 * a + 1);
    const double c =
        wg_weight<V>(variant, hi.nb >= 0 && lo.nb >= 0) * cot[a * n + j];
    if (variant == kFaceVar) {
      if (bc_cot) {
        bc_cot[(2 * a + 1) * n + j] = hi.nb < 0 ? c : 0.0;
        bc_cot[(2 * a) * n + j] = lo.nb < 0 ? -c : 0.0;
      }
    } else {
      if (hi.nb < 0) acc += c;
      if (lo.nb < 0) acc -= c;
    }
  }
  out[j] = acc;
}

}  // namespace
}  // namespace pf

using namespace pf;

#define PF_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) {            \
      set_error(msg);         \
      return PF_ERR_ARG;      \
    }                         \
  } while (0)

extern "C" int pf_wide_grad(const pf_plan *plan, const double *phi,
                            int32_t variant, const double *bc_cells,
                            double *out, void *stream) {
  PF_REQUIRE(plan && phi && out && variant >= 0 && variant <= 2,
             "pf_wide_grad: bad argument");
  PF_REQUIRE(variant != kFaceVar || bc_cells,
             "pf_wide_grad: the face variant needs bc_cells");
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  PF_REQUIRE(!pl.slab, "pf_wide_grad: slab plans are not supported");
  return dispatch(pl, [&](auto v) {
    launch(k_wide_grad<decltype(v)>, grid_for(v.owned()), kBlock,
           static_cast<cudaStream_t>(stream), v, phi, (int)variant, bc_cells,
           out);
    PF_LAUNCH_CHECK("wide_grad");
    return PF_OK;
  });
}

extern "C" int pf_wide_grad_adjoint(const pf_plan *plan, const double *cot,
                                    int32_t variant, double *out,
                                    double *bc_cot, void *stream) {
  PF_REQUIRE(plan && cot && out && variant >= 0 && variant <= 2,
             "pf_wide_grad_adjoint: bad argument");
  const Plan &pl = *reinterpret_cast<const Plan *>(plan);
  PF_REQUIRE(!pl.slab, "pf_wide_grad_adjoint: slab plans are not supported");
  return dispatch(pl, [&](auto v) {
    launch(k_wide_grad_adjoint<decltype(v)>, grid_for(v.owned()), kBlock,
           static_cast<cudaStream_t>(stream), v, cot, (int)variant, out,
           bc_cot);
    PF_LAUNCH_CHECK("wide_grad_adjoint");
    return PF_OK;
  });
}
