// comm.cuh -- slab decomposition over peer memory (NVLink P2P / same device).
//
// A box plan split along axis 0 (the periodic streamwise X of the channel)
// owns nxl planes and carries one ghost plane on each side: the local arrays
// are (nxl + 2) planes long, kernels iterate the owned cells [i0, i1) only and
// read the x-neighbours of the first / last owned plane from the ghost
// planes.  Ranks form a ring (rank - 1 is "left", rank + 1 "right").
//
// Every rank owns one symmetric buffer (cudaMalloc'd at comm creation, the
// same layout on every rank) and maps the buffers of all peers: through
// cudaIpcOpenMemHandle across processes (one process per GPU, NVLink), or
// directly when several slabs share one process and device (tests).  Three
// device-initiated operations move data, all stream ordered and
// host-free, so a solver iteration never returns to the host:
//
//  * allreduce of K doubles, run by the last CTA of every fused reduction
//    (grid_reduce): it stores its K partial totals into slot [rank] of every
//    peer's reduction area, releases a flag there, waits for all peers'
//    flags and sums the G slots in rank order -- bitwise identical on all
//    ranks, no floating-point atomics;
//  * halo exchange: a put kernel stores the first / last owned plane of a
//    set of arrays straight into the left / right neighbour's inbox and
//    releases a flag; a one-thread kernel waits for both flags, then the
//    inbox is copied into the local ghost planes;
//  * barrier (the spectral preconditioner's all-to-all transposes store /
//    load peer spectra directly, separated by barriers).
//
// Flags carry monotonically increasing sequence numbers (never reset), and
// the data areas are double buffered by sequence parity: a rank can only be
// one operation ahead of its slowest peer, so the buffer it writes is never
// the one a peer still reads.  Waits time out (kCommTimeoutNs) into an error
// flag instead of hanging the device.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pf {

constexpr int kMaxRanks = 16;
constexpr int kRedK = 16;              // doubles per rank per allreduce slot
constexpr int kVecRedMax = 4096;       // doubles of the vector allreduce
constexpr int kHaloMaxPlanes = 24;     // component planes per exchange
constexpr int kHaloMaxArrays = 8;
constexpr unsigned long long kCommTimeoutNs = 20ull * 1000 * 1000 * 1000;

// byte offsets inside every rank's symmetric buffer
constexpr int64_t kOffRedFlag = 0;                  // [2][kMaxRanks] u64
constexpr int64_t kOffBarFlag = 512;                // [kMaxRanks] u64
constexpr int64_t kOffHaloFlag = 1024;              // [2][2] u64
constexpr int64_t kOffVecFlag = 1536;               // [2][kMaxRanks] u64
constexpr int64_t kOffRed = 4096;                   // [2][kMaxRanks][kRedK]
constexpr int64_t kOffVec = kOffRed + 2 * kMaxRanks * kRedK * 8;
constexpr int64_t kOffHalo =                        // [2][2][planes][plane]
    kOffVec + 2 * (int64_t)kMaxRanks * kVecRedMax * 8;

// Device-side communicator (lives in device memory; kernels get a pointer).
struct CommDev {
  int32_t rank, world, left, right;
  int64_t plane;          // cells per plane (= ghost plane length)
  int64_t spec_off;       // byte offset of the spectral area
  char *peer[kMaxRanks];  // every rank's symmetric buffer (own at [rank])
  unsigned long long red_seq, halo_seq, bar_seq, vec_seq;
  int32_t err;            // 1: a wait timed out
  unsigned ticket;        // CTA ticket of the halo put
  unsigned long long timeout_ns;
  // first timeout: flag offset in the own buffer, expected and seen value
  long long err_off;
  unsigned long long err_want, err_seen;
};

// component planes of one halo exchange (device view)
struct HaloSet {
  double *comp[kHaloMaxPlanes];  // component base pointers (stride n)
  int32_t planes;
};

// host-side description of one array to exchange
struct HaloItem {
  double *a;      // (ncomp, n) SoA array
  int32_t ncomp;
};

__device__ __forceinline__ unsigned long long ld_acquire(
    const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
               : "=l"(v)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned long long *p,
                                           unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mutable CommDev fields are read / written through volatile accesses: a
// plain load may be served from an SM's L1 line left by an earlier kernel
template <class T>
__device__ __forceinline__ T vload(const T *p) {
  return *reinterpret_cast<const volatile T *>(p);
}
template <class T>
__device__ __forceinline__ void vstore(T *p, T v) {
  *reinterpret_cast<volatile T *>(p) = v;
}

__device__ __forceinline__ unsigned long long *flag_at(char *base,
                                                       int64_t off, int k) {
  return reinterpret_cast<unsigned long long *>(base + off) + k;
}

// spin until *f >= v (or time out into c->err)
__device__ __forceinline__ void wait_flag(CommDev *c,
                                          const unsigned long long *f,
                                          unsigned long long v) {
  if (ld_acquire(f) >= v) return;
  // after a first timeout every later wait fails fast: the host sees the
  // error at its next poll instead of sitting out one timeout per wait
  if (vload(&c->err)) return;
  const unsigned long long t0 = global_ns();
  const unsigned long long lim = c->timeout_ns;
  unsigned long long seen;
  while ((seen = ld_acquire(f)) < v) {
    __nanosleep(64);
    if (global_ns() - t0 > lim) {
      if (!vload(&c->err)) {
        c->err_off = reinterpret_cast<const char *>(f) - c->peer[c->rank];
        c->err_want = v;
        c->err_seen = seen;
      }
      vstore(&c->err, 1);
      return;
    }
  }
}

// Cross-rank allreduce of K values, called by ONE thread (the finaliser of
// a grid reduction).  kMax: maximum instead of sum.
template <int K, bool kMax>
__device__ __forceinline__ void comm_allreduce(CommDev *c, double (&v)[K]) {
  static_assert(K <= kRedK, "allreduce slot too small");
  const unsigned long long e = vload(&c->red_seq) + 1;
  vstore(&c->red_seq, e);
  const int slot = (int)(e & 1);
  const int G = c->world, me = c->rank;
  for (int q = 0; q < G; ++q) {
    double *dst = reinterpret_cast<double *>(c->peer[q] + kOffRed) +
                  ((int64_t)slot * kMaxRanks + me) * kRedK;
#pragma unroll
    for (int k = 0; k < K; ++k) dst[k] = v[k];
  }
  __threadfence_system();
  for (int q = 0; q < G; ++q)
    st_release(flag_at(c->peer[q], kOffRedFlag, slot * kMaxRanks + me), e);
  char *mine = c->peer[me];
  for (int q = 0; q < G; ++q)
    wait_flag(c, flag_at(mine, kOffRedFlag, slot * kMaxRanks + q), e);
  const volatile double *src =
      reinterpret_cast<const double *>(mine + kOffRed) +
      (int64_t)slot * kMaxRanks * kRedK;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double acc = src[k];
    for (int q = 1; q < G; ++q) {
      const double x = src[(int64_t)q * kRedK + k];
      acc = kMax ? fmax(acc, x) : acc + x;
    }
    v[k] = acc;
  }
}

// The communicator of a workspace: its device address sits right after the
// 64 reduction counters at the start of every workspace (null when the plan
// is not distributed).  grid_reduce finds it from the counter pointer.
constexpr int64_t kWsCommOffset = 256;
__device__ __forceinline__ CommDev *ws_comm(const unsigned *counter) {
  return *reinterpret_cast<CommDev *const *>(
      reinterpret_cast<const char *>(counter) + kWsCommOffset);
}

}  // namespace pf
