// plan.cu -- plan lifetime, error reporting, workspace sizing.
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "mg.cuh"

namespace pf {

static thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
thread_local unsigned long long *g_capture_count = nullptr;

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return PF_OK;
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %d (%s) in %s", (int)e,
           cudaGetErrorString(e), what);
  set_error(buf);
  return PF_ERR_CUDA;
}

// the small status reads are stored into the mapped staging buffer by a
// one-CTA kernel, not by a copy engine: a solver's poll then never queues
// behind a caller's bulk device-to-host copy on another stream
__global__ void k_d2h_small(unsigned char *dst, const unsigned char *src,
                            int bytes) {
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

int d2h(const Plan &p, void *host, const void *dev, size_t bytes,
        cudaStream_t s) {
  if (bytes > kPinnedBytes || !p.pinned) {
    set_error("d2h: read too large for the plan's staging buffer");
    return PF_ERR_ARG;
  }
  if (p.pinned_dev && !p.comm) {
    count_launch();
    k_d2h_small<<<1, 128, 0, s>>>(static_cast<unsigned char *>(p.pinned_dev),
                                  static_cast<const unsigned char *>(dev),
                                  (int)bytes);
  } else {
    // slab ranks sharing one device in tests: a copy engine needs no SM
    // while peers' kernels may occupy them all
    PF_CUDA(cudaMemcpyAsync(p.pinned, dev, bytes, cudaMemcpyDeviceToHost, s));
  }
  PF_CUDA(cudaStreamSynchronize(s));
  std::memcpy(host, p.pinned, bytes);
  return PF_OK;
}

}  // namespace pf

using namespace pf;

extern "C" const char *pf_last_error(void) { return g_last_error.c_str(); }

extern "C" int pf_version(void) { return 1; }

extern "C" unsigned long long pf_launch_count(void) { return g_launches.load(); }

extern "C" int pf_plan_create(const pf_plan_desc *desc, pf_plan **out) {
  if (!desc || !out) {
    set_error("pf_plan_create: null argument");
    return PF_ERR_ARG;
  }
  const pf_plan_desc &d = *desc;
  if (d.dim != 2 && d.dim != 3) {
    set_error("pf_plan_create: dim must be 2 or 3");
    return PF_ERR_ARG;
  }
  if (d.n <= 0 || d.n >= (1LL << 26)) {
    set_error("pf_plan_create: cell count out of range (1 .. 2^26-1)");
    return PF_ERR_ARG;
  }
  if (!d.jac || !d.tmat || !d.alpha_diag) {
    set_error("pf_plan_create: missing metrics");
    return PF_ERR_ARG;
  }
  if (d.m > 0 && (!d.bcell || !d.bface || !d.bjac || !d.bt || !d.balpha)) {
    set_error("pf_plan_create: missing boundary arrays");
    return PF_ERR_ARG;
  }
  if (d.topo == PF_TOPO_GATHER) {
    if (!d.nbr) {
      set_error("pf_plan_create: gather topology needs a neighbour table");
      return PF_ERR_ARG;
    }
  } else if (d.topo == PF_TOPO_BOX) {
    int64_t cnt = 1;
    for (int a = 0; a < d.dim; ++a) {
      if (d.box_shape[a] < 1) {
        set_error("pf_plan_create: bad box shape");
        return PF_ERR_ARG;
      }
      cnt *= d.box_shape[a];
    }
    if (cnt != d.n) {
      set_error("pf_plan_create: box shape does not match n");
      return PF_ERR_ARG;
    }
  } else {
    set_error("pf_plan_create: unknown topology");
    return PF_ERR_ARG;
  }
  const bool slab = d.slab_world > 0;
  if (slab) {
    if (d.topo != PF_TOPO_BOX || !d.box_periodic[0] || d.box_shape[0] < 3 ||
        d.slab_world > kMaxRanks || d.slab_rank < 0 ||
        d.slab_rank >= d.slab_world || d.slab_x0 < 0 ||
        d.slab_x0 + d.box_shape[0] - 2 > d.slab_nx) {
      set_error("pf_plan_create: a slab plan needs a box periodic along axis "
                "0 with nxl + 2 planes, 0 <= slab_rank < slab_world <= 16 and "
                "slab_x0 + nxl <= slab_nx");
      return PF_ERR_ARG;
    }
    if (d.has_cross) {
      set_error("pf_plan_create: slab plans support orthogonal grids only");
      return PF_ERR_UNSUPPORTED;
    }
  }
  int dev = 0, sms = 148;
  PF_CUDA(cudaGetDevice(&dev));
  PF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  Plan *p = new Plan();
  p->d = d;
  p->num_sms = sms;
  p->red_blocks = sms * 8 < kMaxRedBlocks ? sms * 8 : kMaxRedBlocks;
  p->slab = slab;
  if (slab) {
    p->plane = d.n / d.box_shape[0];
    p->nxl = d.box_shape[0] - 2;
    p->i0 = (int32_t)p->plane;
    p->i1 = (int32_t)(p->plane * (p->nxl + 1));
    p->ng = (double)d.slab_nx * (double)p->plane;
  } else {
    p->i0 = 0;
    p->i1 = (int32_t)d.n;
    p->ng = (double)d.n;
  }
  p->has_mg = mg_plan(*p, p->mg, &p->mg_bytes);
  {
    const cudaError_t e =
        cudaHostAlloc(&p->pinned, kPinnedBytes, cudaHostAllocMapped);
    if (e != cudaSuccess) {
      delete p;
      return cuda_check(e, "cudaHostAlloc(plan staging)");
    }
    if (cudaHostGetDevicePointer(&p->pinned_dev, p->pinned, 0) != cudaSuccess) {
      cudaGetLastError();
      p->pinned_dev = nullptr;  // copy-engine reads only
    }
  }
  *out = reinterpret_cast<pf_plan *>(p);
  return PF_OK;
}

extern "C" int pf_plan_destroy(pf_plan *plan) {
  Plan *p = reinterpret_cast<Plan *>(plan);
  if (p) {
    if (p->graph.exec) cudaGraphExecDestroy(p->graph.exec);
    if (p->graph.cap) cudaStreamDestroy(p->graph.cap);
    if (p->pinned) cudaFreeHost(p->pinned);
  }
  delete p;
  return PF_OK;
}

extern "C" int64_t pf_workspace_bytes(const pf_plan *plan) {
  if (!plan) return -1;
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  return workspace_bytes(p.d.n, p.d.dim);
}

extern "C" int64_t pf_mg_workspace_bytes(const pf_plan *plan) {
  if (!plan) return -1;
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  return p.has_mg ? p.mg_bytes : 0;
}

extern "C" int pf_mg_levels(const pf_plan *plan) {
  if (!plan) return -1;
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  return p.has_mg ? p.mg.nlev : 0;
}

extern "C" int pf_mg_kind(const pf_plan *plan) {
  if (!plan) return PF_GEOM_NONE;
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  if (!p.has_mg) return PF_GEOM_NONE;
  return p.mg.spectral ? PF_GEOM_SPECTRAL : PF_GEOM_MULTIGRID;
}

extern "C" int pf_mg_setup(const pf_plan *plan, const double *k,
                           void *mg_workspace, void *stream) {
  if (!plan || !k || !mg_workspace) {
    set_error("pf_mg_setup: null argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  if (!p.has_mg) {
    set_error("pf_mg_setup: multigrid is not available for this plan");
    return PF_ERR_UNSUPPORTED;
  }
  MgHierarchy h = p.mg;
  mg_bind(h, mg_workspace);
  return mg_setup(h, k, p.d.n, static_cast<cudaStream_t>(stream), nullptr,
                  &p);
}
