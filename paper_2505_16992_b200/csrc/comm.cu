// comm.cu -- slab communicator: symmetric buffers, halo exchange, barrier,
// vector allreduce (see comm.cuh).
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "mg.cuh"
#include "spectral.cuh"

namespace pf {

// ---------------------------------------------------------------------------
// halo exchange

// element t of the put: side 0 sends my first owned plane to the left
// neighbour's HI inbox, side 1 my last owned plane to the right neighbour's
// LO inbox
__global__ void __launch_bounds__(kBlock)
    k_halo_put(CommDev *c, HaloSet hs, int64_t n, int64_t nxl) {
  const int64_t plane = c->plane;
  const unsigned long long e = vload(&c->halo_seq) + 1;
  const int par = (int)(e & 1);
  const int64_t per_side = (int64_t)hs.planes * plane;
  const int64_t total = 2 * per_side;
  char *lbase = c->peer[c->left], *rbase = c->peer[c->right];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int side = t >= per_side;
    const int64_t r = t - side * per_side;
    const int k = (int)(r / plane);
    const int64_t el = r - (int64_t)k * plane;
    const double *src = hs.comp[k] + (side ? nxl : 1) * plane + el;
    (void)n;
    // LO = 0, HI = 1: the half of the receiver's inbox feeding that ghost
    const int dst_half = side ? 0 : 1;
    char *base = side ? rbase : lbase;
    double *dst = reinterpret_cast<double *>(base + kOffHalo) +
                  (((int64_t)par * 2 + dst_half) * kHaloMaxPlanes + k) * plane +
                  el;
    *dst = *src;
  }
  // every thread fences its own peer stores before the CTA's ticket
  __threadfence_system();
  // last CTA out releases the flags
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned t = atomicAdd(&c->ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    st_release(flag_at(lbase, kOffHaloFlag, par * 2 + 1), e);
    st_release(flag_at(rbase, kOffHaloFlag, par * 2 + 0), e);
    vstore(&c->halo_seq, e);
    vstore(&c->ticket, 0u);
  }
}

// one thread waits for both neighbours' flags of the current exchange (a
// single spinning CTA: several slabs sharing a device must never fill it
// with waiting CTAs)
__global__ void k_halo_wait(CommDev *c) {
  if (threadIdx.x != 0) return;
  const unsigned long long e = vload(&c->halo_seq);
  const int par = (int)(e & 1);
  char *mine = c->peer[c->rank];
  wait_flag(c, flag_at(mine, kOffHaloFlag, par * 2 + 0), e);
  wait_flag(c, flag_at(mine, kOffHaloFlag, par * 2 + 1), e);
  __threadfence();
}

// inbox -> ghost planes (after k_halo_wait)
__global__ void __launch_bounds__(kBlock)
    k_halo_unpack(CommDev *c, HaloSet hs, int64_t nxl) {
  const int64_t plane = c->plane;
  const int par = (int)(vload(&c->halo_seq) & 1);
  const double *inbox =
      reinterpret_cast<const double *>(c->peer[c->rank] + kOffHalo);
  const int64_t per_side = (int64_t)hs.planes * plane;
  const int64_t total = 2 * per_side;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int side = t >= per_side;  // 0: lo ghost, 1: hi ghost
    const int64_t r = t - side * per_side;
    const int k = (int)(r / plane);
    const int64_t el = r - (int64_t)k * plane;
    const double v = __ldcv(inbox + (((int64_t)par * 2 + side) * kHaloMaxPlanes +
                                     k) * plane + el);
    hs.comp[k][(side ? nxl + 1 : 0) * plane + el] = v;
  }
}

// ---------------------------------------------------------------------------
// barrier and vector allreduce (one CTA)

__global__ void k_comm_barrier(CommDev *c) {
  if (threadIdx.x != 0) return;
  const unsigned long long e = vload(&c->bar_seq) + 1;
  vstore(&c->bar_seq, e);
  __threadfence_system();
  for (int q = 0; q < c->world; ++q)
    st_release(flag_at(c->peer[q], kOffBarFlag, c->rank), e);
  for (int q = 0; q < c->world; ++q)
    wait_flag(c, flag_at(c->peer[c->rank], kOffBarFlag, q), e);
  __threadfence_system();
}

// buf[0..k) <- sum (op 0) / max (op 1) over ranks, in rank order
__global__ void __launch_bounds__(1024)
    k_comm_vec_allreduce(CommDev *c, double *buf, int k, int op) {
  __shared__ unsigned long long e;
  const int G = c->world, me = c->rank;
  if (threadIdx.x == 0) {
    e = vload(&c->vec_seq) + 1;
    vstore(&c->vec_seq, e);
  }
  __syncthreads();
  const int slot = (int)(e & 1);
  for (int q = 0; q < G; ++q) {
    double *dst = reinterpret_cast<double *>(c->peer[q] + kOffVec) +
                  ((int64_t)slot * kMaxRanks + me) * kVecRedMax;
    for (int j = threadIdx.x; j < k; j += blockDim.x) dst[j] = buf[j];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < G; ++q)
      st_release(flag_at(c->peer[q], kOffVecFlag, slot * kMaxRanks + me), e);
    for (int q = 0; q < G; ++q)
      wait_flag(c, flag_at(c->peer[me], kOffVecFlag, slot * kMaxRanks + q),
                e);
    __threadfence();
  }
  __syncthreads();
  const double *src = reinterpret_cast<const double *>(c->peer[me] + kOffVec) +
                      (int64_t)slot * kMaxRanks * kVecRedMax;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double acc = __ldcv(src + j);
    for (int q = 1; q < G; ++q) {
      const double x = __ldcv(src + (int64_t)q * kVecRedMax + j);
      acc = op ? fmax(acc, x) : acc + x;
    }
    buf[j] = acc;
  }
}

// ---------------------------------------------------------------------------
// host helpers used by the other translation units

int halo_exchange(const Plan &p, const HaloItem *items, int count,
                  cudaStream_t s) {
  if (!p.comm) return PF_OK;
  HaloSet hs{};
  int planes = 0;
  for (int j = 0; j < count; ++j) {
    if (!items[j].a) continue;
    for (int q = 0; q < items[j].ncomp; ++q) {
      if (planes >= kHaloMaxPlanes) {
        set_error("halo_exchange: too many component planes");
        return PF_ERR_ARG;
      }
      hs.comp[planes++] = items[j].a + (int64_t)q * p.d.n;
    }
  }
  if (!planes) return PF_OK;
  hs.planes = planes;
  const int64_t plane = p.comm->plane;
  const int64_t total = 2 * planes * plane;
  const int g = (int)std::min<int64_t>(grid_for(total), p.num_sms * 4);
  launch(k_halo_put, g, kBlock, s, p.comm->dev, hs, p.d.n, p.comm->nxl);
  launch(k_halo_wait, 1, 32, s, p.comm->dev);
  const int gg = (int)std::min<int64_t>(grid_for(total), p.num_sms * 4);
  launch(k_halo_unpack, gg, kBlock, s, p.comm->dev, hs, p.comm->nxl);
  PF_LAUNCH_CHECK("halo exchange");
  return PF_OK;
}

int comm_check(const Plan &p, cudaStream_t s) {
  if (!p.comm) return PF_OK;
  int32_t err = 0;
  int rc = d2h(p, &err, &p.comm->dev->err, sizeof(err), s);
  if (rc) return rc;
  if (err)
    return pf_comm_status(reinterpret_cast<const pf_comm *>(p.comm), s);
  return PF_OK;
}

int comm_barrier(const Plan &p, cudaStream_t s) {
  if (!p.comm) return PF_OK;
  launch(k_comm_barrier, 1, 32, s, p.comm->dev);
  PF_LAUNCH_CHECK("comm barrier");
  return PF_OK;
}

int comm_vec_allreduce(const Plan &p, double *buf, int k, int op,
                       cudaStream_t s) {
  if (!p.comm) return PF_OK;
  if (k > kVecRedMax) {
    set_error("comm_vec_allreduce: vector too long");
    return PF_ERR_ARG;
  }
  launch(k_comm_vec_allreduce, 1, 1024, s, p.comm->dev, buf, k, op);
  PF_LAUNCH_CHECK("comm vec allreduce");
  return PF_OK;
}

int comm_vec_allreduce_n(const Plan &p, double *buf, int64_t k, int op,
                         cudaStream_t s) {
  for (int64_t off = 0; off < k; off += kVecRedMax) {
    const int len = (int)std::min<int64_t>(kVecRedMax, k - off);
    int rc = comm_vec_allreduce(p, buf + off, len, op, s);
    if (rc) return rc;
  }
  return PF_OK;
}

}  // namespace pf

// ===========================================================================
// C ABI

using namespace pf;

extern "C" int pf_comm_create(const pf_plan *plan, pf_comm **out) {
  if (!plan || !out) {
    set_error("pf_comm_create: null argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  if (!p.slab) {
    set_error("pf_comm_create: the plan is not a slab plan "
              "(pf_plan_desc.slab_world == 0)");
    return PF_ERR_ARG;
  }
  CommHost *c = new CommHost();
  c->rank = p.d.slab_rank;
  c->world = p.d.slab_world;
  c->plane = p.plane;
  c->nxl = p.nxl;
  c->spec_bytes = p.has_mg && p.mg.spectral ? spec_slab_bytes(p.mg.sp) : 0;
  c->sym_bytes = kOffHalo + 2 * 2 * (int64_t)kHaloMaxPlanes * c->plane * 8;
  c->spec_off = (c->sym_bytes + 4095) / 4096 * 4096;
  c->sym_bytes = c->spec_off + c->spec_bytes;
  int rc = cuda_check(cudaMalloc(&c->sym, c->sym_bytes), "cudaMalloc(sym)");
  if (!rc) rc = cuda_check(cudaMemset(c->sym, 0, c->sym_bytes), "memset(sym)");
  if (!rc) rc = cuda_check(cudaMalloc(&c->dev, sizeof(CommDev)), "cudaMalloc(comm)");
  if (!rc) rc = cuda_check(cudaMallocHost(&c->pinned, sizeof(CommDev)),
                           "cudaMallocHost(comm staging)");
  if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "comm create sync");
  if (rc) {
    if (c->sym) cudaFree(c->sym);
    if (c->dev) cudaFree(c->dev);
    if (c->pinned) cudaFreeHost(c->pinned);
    delete c;
    return rc;
  }
  std::memset(&c->host, 0, sizeof(CommDev));
  c->host.rank = c->rank;
  c->host.world = c->world;
  c->host.left = (c->rank + c->world - 1) % c->world;
  c->host.right = (c->rank + 1) % c->world;
  c->host.plane = c->plane;
  c->host.spec_off = c->spec_off;
  c->host.peer[c->rank] = static_cast<char *>(c->sym);
  c->host.timeout_ns = kCommTimeoutNs;
  if (const char *e = getenv("PF_COMM_TIMEOUT_S")) {
    const double sec = atof(e);
    if (sec > 0) c->host.timeout_ns = (unsigned long long)(sec * 1e9);
  }
  *out = reinterpret_cast<pf_comm *>(c);
  return PF_OK;
}

extern "C" int pf_comm_ipc_handle(const pf_comm *comm, void *handle_host) {
  if (!comm || !handle_host) {
    set_error("pf_comm_ipc_handle: null argument");
    return PF_ERR_ARG;
  }
  const CommHost *c = reinterpret_cast<const CommHost *>(comm);
  cudaIpcMemHandle_t h;
  PF_CUDA(cudaIpcGetMemHandle(&h, c->sym));
  std::memcpy(handle_host, &h, sizeof(h));
  return PF_OK;
}

extern "C" int pf_comm_open_peer(pf_comm *comm, int32_t peer,
                                 const void *handle_host) {
  CommHost *c = reinterpret_cast<CommHost *>(comm);
  if (!c || !handle_host || peer < 0 || peer >= c->world || peer == c->rank) {
    set_error("pf_comm_open_peer: bad argument");
    return PF_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle_host, sizeof(h));
  void *ptr = nullptr;
  PF_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
  c->host.peer[peer] = static_cast<char *>(ptr);
  c->ipc_opened[peer] = true;
  return PF_OK;
}

extern "C" int pf_comm_set_local_peer(pf_comm *comm, int32_t peer,
                                      const pf_comm *other) {
  CommHost *c = reinterpret_cast<CommHost *>(comm);
  const CommHost *o = reinterpret_cast<const CommHost *>(other);
  if (!c || !o || peer < 0 || peer >= c->world || o->rank != peer ||
      o->sym_bytes != c->sym_bytes) {
    set_error("pf_comm_set_local_peer: bad argument");
    return PF_ERR_ARG;
  }
  c->host.peer[peer] = static_cast<char *>(o->sym);
  return PF_OK;
}

extern "C" int64_t pf_comm_bytes(const pf_comm *comm) {
  const CommHost *c = reinterpret_cast<const CommHost *>(comm);
  return c ? c->sym_bytes : -1;
}

extern "C" int pf_plan_attach_comm(pf_plan *plan, pf_comm *comm,
                                   void *workspace, void *stream) {
  if (!plan || !comm || !workspace) {
    set_error("pf_plan_attach_comm: null argument");
    return PF_ERR_ARG;
  }
  Plan &p = *reinterpret_cast<Plan *>(plan);
  CommHost *c = reinterpret_cast<CommHost *>(comm);
  for (int q = 0; q < c->world; ++q) {
    if (!c->host.peer[q]) {
      set_error("pf_plan_attach_comm: peer buffer " + std::to_string(q) +
                " not mapped (pf_comm_open_peer / pf_comm_set_local_peer)");
      return PF_ERR_ARG;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PF_CUDA(cudaMemcpyAsync(c->dev, &c->host, sizeof(CommDev),
                          cudaMemcpyHostToDevice, s));
  PF_CUDA(cudaMemcpyAsync(static_cast<char *>(workspace) + kWsCommOffset,
                          &c->dev, sizeof(CommDev *), cudaMemcpyHostToDevice,
                          s));
  PF_CUDA(cudaStreamSynchronize(s));
  p.comm = c;
  if (p.has_mg && p.mg.spectral) spec_slab_bind(p.mg.sp, *c);
  return PF_OK;
}

extern "C" int pf_comm_status(const pf_comm *comm, void *stream) {
  const CommHost *c = reinterpret_cast<const CommHost *>(comm);
  if (!c) {
    set_error("pf_comm_status: null argument");
    return PF_ERR_ARG;
  }
  CommDev d;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PF_CUDA(cudaMemcpyAsync(c->pinned, c->dev, sizeof(d),
                          cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
  std::memcpy(&d, c->pinned, sizeof(d));
  if (d.err) {
    const char *what = d.err_off < kOffBarFlag    ? "allreduce"
                       : d.err_off < kOffHaloFlag ? "barrier"
                       : d.err_off < kOffVecFlag  ? "halo"
                                                  : "vector allreduce";
    set_error("slab communicator (rank " + std::to_string(d.rank) +
              "): a peer wait timed out in a " + what + " (flag offset " +
              std::to_string(d.err_off) + ", wanted " +
              std::to_string(d.err_want) + ", saw " +
              std::to_string(d.err_seen) + "; sequence red " +
              std::to_string(d.red_seq) + " halo " +
              std::to_string(d.halo_seq) + " bar " +
              std::to_string(d.bar_seq) + " vec " +
              std::to_string(d.vec_seq) + ")");
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

extern "C" int pf_comm_destroy(pf_comm *comm) {
  CommHost *c = reinterpret_cast<CommHost *>(comm);
  if (!c) return PF_OK;
  for (int q = 0; q < c->world; ++q)
    if (c->ipc_opened[q]) cudaIpcCloseMemHandle(c->host.peer[q]);
  if (c->dev) cudaFree(c->dev);
  if (c->sym) cudaFree(c->sym);
  if (c->pinned) cudaFreeHost(c->pinned);
  delete c;
  return PF_OK;
}

extern "C" int pf_halo_exchange(const pf_plan *plan, const uint64_t *arrays_host,
                                const int32_t *ncomp_host, int32_t count,
                                void *stream) {
  if (!plan || (count > 0 && (!arrays_host || !ncomp_host)) || count < 0 ||
      count > kHaloMaxArrays) {
    set_error("pf_halo_exchange: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  HaloItem it[kHaloMaxArrays];
  for (int j = 0; j < count; ++j)
    it[j] = HaloItem{reinterpret_cast<double *>(arrays_host[j]), ncomp_host[j]};
  return halo_exchange(p, it, count, static_cast<cudaStream_t>(stream));
}

extern "C" int pf_comm_allreduce(const pf_plan *plan, double *buf, int32_t k,
                                 int32_t op, void *stream) {
  if (!plan || !buf || k < 0 || op < 0 || op > 1) {
    set_error("pf_comm_allreduce: bad argument");
    return PF_ERR_ARG;
  }
  const Plan &p = *reinterpret_cast<const Plan *>(plan);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int off = 0; off < k; off += kVecRedMax) {
    int rc = comm_vec_allreduce(p, buf + off, std::min(kVecRedMax, k - off),
                                op, s);
    if (rc) return rc;
  }
  return PF_OK;
}

extern "C" int pf_comm_barrier(const pf_plan *plan, void *stream) {
  if (!plan) {
    set_error("pf_comm_barrier: null argument");
    return PF_ERR_ARG;
  }
  return comm_barrier(*reinterpret_cast<const Plan *>(plan),
                      static_cast<cudaStream_t>(stream));
}

extern "C" int pf_comm_counters(const pf_comm *comm, uint64_t *out4_host,
                                void *stream) {
  const CommHost *c = reinterpret_cast<const CommHost *>(comm);
  if (!c || !out4_host) {
    set_error("pf_comm_counters: null argument");
    return PF_ERR_ARG;
  }
  CommDev d;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PF_CUDA(cudaMemcpyAsync(c->pinned, c->dev, sizeof(d),
                          cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
  std::memcpy(&d, c->pinned, sizeof(d));
  out4_host[0] = d.red_seq;
  out4_host[1] = d.halo_seq;
  out4_host[2] = d.bar_seq;
  out4_host[3] = d.vec_seq;
  return PF_OK;
}
