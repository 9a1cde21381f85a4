// spectral.cu -- FFT / tridiagonal preconditioner (see spectral.cuh).
#include <algorithm>
#include <cstdlib>

#include "mg.cuh"
#include "spectral.cuh"

namespace pf {

constexpr int kFftThreads = 256;
constexpr int kFftElems = 1024;  // complex elements per CTA buffer (16 KB)
constexpr int kYThreads = 128;
constexpr int kMaxLines = 2 * kFftElems / 4;  // real Z lines per tile (N >= 4)

#define SPEC_DONE_RETURN \
  if (done && *done) return

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <bool kInv>
__device__ __forceinline__ double2 twiddle(const double2 *tw, int k) {
  double2 w = __ldg(tw + k);
  if (kInv) w.y = -w.y;
  return w;
}

// Shared-memory layout of a line: element i sits at pad(i) = i + i / 16, so
// the power-of-two strides of the butterflies spread over the banks (one
// 16-byte pad slot per 16 elements; line stride padded_len(N)).
__host__ __device__ constexpr int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int n) {
  return n + (n >> 4);
}

// Stockham autosort FFT (radix 4, a final radix-2 stage when log2 N is odd)
// of `nl` lines of length N held in shared memory (padded layout above);
// b is scratch of the same size.  Returns the buffer holding the natural-order
// result.  Forward: exp(-2 pi i jk / N); inverse: exp(+...), unnormalised.
template <bool kInv>
__device__ double2 *fft_lines(double2 *a, double2 *b, int N, int nl,
                              const double2 *tw) {
  const int q4 = N >> 2, lg = __ffs(N) - 1;
  const int NP = padded_len(N);
  int n = N, ls = 0;  // current length, log2 of the stride
  while (n >= 4) {
    const int n1 = n >> 2, s = 1 << ls;
    for (int t = threadIdx.x; t < nl * q4; t += blockDim.x) {
      const int line = t >> (lg - 2);
      const int k = t & (q4 - 1);
      const int q = k & (s - 1), p = k >> ls;
      const double2 *x = a + line * NP;
      double2 *y = b + line * NP;
      const double2 x0 = x[pad(q + s * p)], x1 = x[pad(q + s * (p + n1))];
      const double2 x2 = x[pad(q + s * (p + 2 * n1))];
      const double2 x3 = x[pad(q + s * (p + 3 * n1))];
      const double2 apc = cadd(x0, x2), amc = csub(x0, x2);
      const double2 bpd = cadd(x1, x3), bmd = csub(x1, x3);
      // forward: j (b - d) with j = i; the inverse flips its sign
      const double2 jb = kInv ? make_double2(bmd.y, -bmd.x)
                              : make_double2(-bmd.y, bmd.x);
      const int ps = p << ls;
      y[pad(q + s * (4 * p))] = cadd(apc, bpd);
      y[pad(q + s * (4 * p + 1))] = cmul(twiddle<kInv>(tw, ps), csub(amc, jb));
      y[pad(q + s * (4 * p + 2))] =
          cmul(twiddle<kInv>(tw, 2 * ps), csub(apc, bpd));
      y[pad(q + s * (4 * p + 3))] =
          cmul(twiddle<kInv>(tw, 3 * ps), cadd(amc, jb));
    }
    __syncthreads();
    double2 *tmp = a;
    a = b;
    b = tmp;
    n >>= 2;
    ls += 2;
  }
  if (n == 2) {
    const int s = N >> 1;
    for (int t = threadIdx.x; t < nl * s; t += blockDim.x) {
      const int line = t >> (lg - 1);
      const int q = t & (s - 1);
      const double2 *x = a + line * NP;
      double2 *y = b + line * NP;
      const double2 x0 = x[pad(q)], x1 = x[pad(q + s)];
      y[pad(q)] = cadd(x0, x1);
      y[pad(q + s)] = csub(x0, x1);
    }
    __syncthreads();
    a = b;
  }
  return a;
}

// The Z passes handle the real Z lines l0 .. l0 + 2 LP - 1 of a tile (lines
// enumerated X fastest, then Y; slab plans skip the ghost plane at local
// X = 0).  Their first elements and (x, y) are tabulated once per tile, so
// the element loops carry no integer division.
template <int N>
struct ZLinesT {
  int32_t base[N];
  int32_t x[N], y[N];
};
using ZLines = ZLinesT<kMaxLines>;

template <class T>
__device__ __forceinline__ void zlines_fill(const SpecPlan &sp, int32_t l0,
                                            int nl, T &t) {
  const int32_t last = sp.nxl * sp.sy - 1;
  for (int j = threadIdx.x; j < nl; j += blockDim.x) {
    const int32_t l = min(l0 + j, last);
    const int32_t x = l % sp.nxl, y = l / sp.nxl;
    t.base[j] = ((x + sp.xoff) * sp.sy + y) * sp.sz;
    t.x[j] = x;
    t.y[j] = y;
  }
}

// rank holding wavenumber kz of the transposed spectrum
__device__ __forceinline__ int kz_owner(const SpecPlan &sp, int kz) {
  int q = 0;
  while (kz >= sp.kz0[q + 1]) ++q;
  return q;
}

// address of (line (x, y), wavenumber kz) in the owner's transposed
// spectrum (Y, kz - kz0[q], global X): a peer address when another rank
// owns kz
__device__ __forceinline__ double2 *spec_at(const SpecPlan &sp, int32_t x,
                                            int32_t y, int kz) {
  const int q = kz_owner(sp, kz);
  const int nkq = sp.kz0[q + 1] - sp.kz0[q];
  return sp.peer_s[q] + ((int64_t)y * nkq + (kz - sp.kz0[q])) * sp.sx +
         sp.x0 + x;
}
// one GPU: every wavenumber is local (no owner search, so the loads of an
// unrolled loop issue back to back)
template <bool kSlab>
__device__ __forceinline__ double2 *spec_at_t(const SpecPlan &sp, int32_t x,
                                              int32_t y, int kz) {
  if (kSlab) return spec_at(sp, x, y, kz);
  return sp.s + ((int64_t)y * sp.nkz + kz) * sp.sx + x;
}

// pass 1: real FFT along Z, two real lines per complex transform
__global__ void __launch_bounds__(kFftThreads)
    k_spec_fwd_z(SpecPlan sp, const double *__restrict__ r, const int *done) {
  SPEC_DONE_RETURN;
  extern __shared__ double2 sm[];
  __shared__ ZLines zl;
  const int N = sp.sz, LP = sp.lpz, nk = sp.nkz, NP = padded_len(N);
  const int lg = __ffs(N) - 1, lg2p = __ffs(2 * LP) - 1;
  const int32_t npairs = sp.nxl * sp.sy / 2;
  const int32_t ntiles = (npairs + LP - 1) / LP;
  for (int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t g0 = tile * LP;
    zlines_fill(sp, 2 * g0, 2 * LP, zl);
    __syncthreads();
    for (int e = threadIdx.x; e < LP * N; e += blockDim.x) {
      const int j = e >> lg, z = e & (N - 1);
      double2 v = make_double2(0.0, 0.0);
      if (g0 + j < npairs) {
        v.x = r[zl.base[2 * j] + z];
        v.y = r[zl.base[2 * j + 1] + z];
      }
      sm[j * NP + pad(z)] = v;
    }
    __syncthreads();
    const double2 *f = fft_lines<false>(sm, sm + LP * NP, N, LP, sp.twz);
    for (int e = threadIdx.x; e < 2 * LP * nk; e += blockDim.x) {
      const int kz = e >> lg2p, jj = e & (2 * LP - 1);
      const int j = jj >> 1, side = jj & 1;
      if (g0 + j >= npairs) continue;
      const double2 zk = f[j * NP + pad(kz)];
      const double2 zm = f[j * NP + pad((N - kz) & (N - 1))];
      // Z = A + iB with A, B the transforms of the two real lines
      const double2 o =
          side == 0 ? make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y))
                    : make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
      // slab plans: the transpose to the kz owner happens here, as a
      // store into the peer's spectrum over NVLink
      *spec_at(sp, zl.x[jj], zl.y[jj], kz) = o;
    }
    __syncthreads();
  }
}

// passes 2 / 4: complex FFT along X, in place on the work array
template <bool kInv>
__global__ void __launch_bounds__(kFftThreads)
    k_spec_x(SpecPlan sp, const int *done) {
  SPEC_DONE_RETURN;
  extern __shared__ double2 sm[];
  const int N = sp.sx, LP = sp.lpx, NP = padded_len(N), lg = __ffs(N) - 1;
  const int64_t nlines =
      (int64_t)sp.sy * (sp.kz0[sp.rank + 1] - sp.kz0[sp.rank]);
  const int64_t ntiles = (nlines + LP - 1) / LP;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t l0 = tile * LP;
    const int64_t nl = nlines - l0 < LP ? nlines - l0 : LP;
    double2 *src = sp.s + l0 * N;
    for (int e = threadIdx.x; e < LP * N; e += blockDim.x) {
      const int ln = e >> lg, xx = e & (N - 1);
      sm[ln * NP + pad(xx)] =
          e < nl * N ? __ldcg(src + e) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double2 *f = fft_lines<kInv>(sm, sm + LP * NP, N, LP, sp.twx);
    for (int e = threadIdx.x; e < nl * N; e += blockDim.x) {
      const int ln = e >> lg, xx = e & (N - 1);
      src[e] = f[ln * NP + pad(xx)];
    }
    __syncthreads();
  }
}

// setup: the Thomas factors of every wavenumber pair's Y system (they
// depend on the plane-mean weights only, so once per operator, not per
// application): c'_y and 1 / den_y, one thread per column
__global__ void __launch_bounds__(kYThreads)
    k_spec_factors(SpecPlan sp, const int *done) {
  SPEC_DONE_RETURN;
  extern __shared__ double sh[];
  const int sy = sp.sy;
  double *ax = sh, *ay = sh + sy, *az = sh + 2 * sy;
  for (int y = threadIdx.x; y < sy; y += blockDim.x) {
    ax[y] = sp.ax[y];
    ay[y] = y + 1 < sy ? sp.ay[y] : 0.0;
    az[y] = sp.az[y];
  }
  __syncthreads();
  const int kzb = sp.kz0[sp.rank];
  const int64_t ncol = (int64_t)(sp.kz0[sp.rank + 1] - kzb) * sp.sx;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncol) return;
  const int kx = (int)(col % sp.sx), kz = kzb + (int)(col / sp.sx);
  const double lxv = sp.lx[kx], lzv = sp.lz[kz];
  const bool pinned = kz == 0 && kx == 0;
  double cprev = 0.0;
  for (int y = 0; y < sy; ++y) {
    const double lo = y > 0 ? ay[y - 1] : 0.0, up = ay[y];
    double c = 0.0, iv = 0.0;
    if (!(pinned && y == sy - 1)) {
      const double den = ax[y] * lxv + az[y] * lzv + lo + up + lo * cprev;
      iv = 1.0 / den;
      c = -up * iv;
    }
    cprev = c;
    sp.cw[(int64_t)y * ncol + col] = c;
    sp.iw[(int64_t)y * ncol + col] = iv;
  }
}

// pass 3: per wavenumber pair (kx, kz) the tridiagonal Y system
//   (ax lx + az lz + ay- + ay+) z_y - ay- z_{y-1} - ay+ z_{y+1} = rhs_y,
// one thread per real / imaginary part (the coefficients are real), with
// the factors of k_spec_factors: no division on the sweeps' dependency
// chain.  The forward sweep overwrites the work array in place.  The
// 1 / (sx sz) normalisation of the transforms is folded in here.
__global__ void __launch_bounds__(kYThreads)
    k_spec_ysolve(SpecPlan sp, const int *done) {
  SPEC_DONE_RETURN;
  extern __shared__ double sh[];
  const int sy = sp.sy;
  double *ax = sh, *ay = sh + sy, *az = sh + 2 * sy;
  for (int y = threadIdx.x; y < sy; y += blockDim.x) {
    ax[y] = sp.ax[y];
    ay[y] = y + 1 < sy ? sp.ay[y] : 0.0;
    az[y] = sp.az[y];
  }
  __syncthreads();
  const int kzb = sp.kz0[sp.rank];
  const int64_t ncol = (int64_t)(sp.kz0[sp.rank + 1] - kzb) * sp.sx;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = t < 2 * ncol;
  const int64_t col = t >> 1;
  const int comp = (int)(t & 1);
  const int kx = (int)(col % sp.sx), kz = kzb + (int)(col / sp.sx);
  const bool pinned = kz == 0 && kx == 0;
  const double scale = 1.0 / ((double)sp.sx * sp.sz);
  double *sv = reinterpret_cast<double *>(sp.s);
  const int64_t ystride = 2 * ncol;
  constexpr int C = 16;
  (void)comp;
  if (active) {
    double dp = 0.0;
    for (int y0 = 0; y0 < sy; y0 += C) {
      double rr[C], ivs[C];
#pragma unroll
      for (int k = 0; k < C; ++k)
        if (y0 + k < sy) {
          rr[k] = __ldcg(sv + (int64_t)(y0 + k) * ystride + t);
          ivs[k] = __ldcg(sp.iw + (int64_t)(y0 + k) * ncol + col);
        }
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int y = y0 + k;
        if (y >= sy) break;
        const double lo = y > 0 ? ay[y - 1] : 0.0;
        dp = (pinned && y == sy - 1) ? 0.0
                                     : (rr[k] * scale + lo * dp) * ivs[k];
        sv[(int64_t)y * ystride + t] = dp;
      }
    }
  }
  if (active) {
    double zn = 0.0;
    for (int y0 = sy - 1; y0 >= 0; y0 -= C) {
      double dd[C], cc[C];
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int y = y0 - k;
        if (y >= 0) {
          dd[k] = sv[(int64_t)y * ystride + t];
          cc[k] = __ldcg(sp.cw + (int64_t)y * ncol + col);
        }
      }
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int y = y0 - k;
        if (y < 0) break;
        zn = dd[k] - cc[k] * zn;
        sv[(int64_t)y * ystride + t] = zn;
      }
    }
  }
}

// pass 5: inverse real FFT along Z (two lines per complex transform), z
// written in the cell layout; optionally the CG z-sums and beta
template <bool kSums>
__global__ void __launch_bounds__(kFftThreads)
    k_spec_inv_z(SpecPlan sp, const double *__restrict__ r,
                 double *__restrict__ z, CgFuse fz, const int *done) {
  SPEC_DONE_RETURN;
  extern __shared__ double2 sm[];
  __shared__ ZLines zl;
  const int N = sp.sz, LP = sp.lpz, half = N >> 1, NP = padded_len(N);
  const int lg = __ffs(N) - 1, lgp = __ffs(LP) - 1;
  const int32_t npairs = sp.nxl * sp.sy / 2;
  const int32_t ntiles = (npairs + LP - 1) / LP;
  double sums[3] = {0.0, 0.0, 0.0};
  for (int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t g0 = tile * LP;
    zlines_fill(sp, 2 * g0, 2 * LP, zl);
    __syncthreads();
    for (int e = threadIdx.x; e < LP * N; e += blockDim.x) {
      const int k = e >> lgp, j = e & (LP - 1);
      double2 v = make_double2(0.0, 0.0);
      if (g0 + j < npairs) {
        const int kk = k <= half ? k : N - k;
        // slab plans: the inverse transpose, loads from the kz owner
        const double2 a =
            __ldcg(spec_at(sp, zl.x[2 * j], zl.y[2 * j], kk));
        const double2 b =
            __ldcg(spec_at(sp, zl.x[2 * j + 1], zl.y[2 * j + 1], kk));
        v = k <= half ? make_double2(a.x - b.y, a.y + b.x)
                      : make_double2(a.x + b.y, b.x - a.y);
      }
      sm[j * NP + pad(k)] = v;
    }
    __syncthreads();
    const double2 *f = fft_lines<true>(sm, sm + LP * NP, N, LP, sp.twz);
    for (int e = threadIdx.x; e < LP * N; e += blockDim.x) {
      const int j = e >> lg, zz = e & (N - 1);
      if (g0 + j >= npairs) continue;
      const double2 v = f[j * NP + pad(zz)];
      const int32_t i0 = zl.base[2 * j] + zz;
      const int32_t i1 = zl.base[2 * j + 1] + zz;
      z[i0] = v.x;
      z[i1] = v.y;
      if (kSums) {
        const double r0 = r[i0], r1 = r[i1];
        sums[0] += v.x + v.y;
        sums[1] += r0 * v.x + r1 * v.y;
        sums[2] += r0 + r1;
      }
    }
    __syncthreads();
  }
  if (kSums) {
    double tot[3];
    if (grid_reduce<3>(sums, fz.partials, fz.counter, tot))
      cg_fin_z(fz.st, tot[0], tot[1], tot[2], sp.sx * sp.sy * sp.sz,
               fz.initial != 0);
  }
}

// ---------------------------------------------------------------------------
// Length-256 transforms (the channel's X and Z): four-step FFT 256 = 16 x 16
// in registers.  A line is owned by 16 threads; thread c holds x[16 n1 + c],
// transforms over n1 in registers (radix 4 x 4), applies W256^(c k1),
// exchanges through one padded shared-memory transpose, and transforms over
// n2.  Two shared-memory passes per transform instead of the Stockham
// kernel's eight, no per-butterfly twiddle loads, and 16 independent loads
// in flight per thread.

constexpr int kR = 16, kN16 = kR * kR;
constexpr int kL16 = 8;             // complex lines per CTA
constexpr int kT16 = kL16 * kR;     // threads per CTA
// natural-order line stride: padded_len(256) + 1, odd in 16-byte units so
// the 8 lines of a tile read at one wavenumber fall in distinct banks
constexpr int kLP16 = padded_len(kN16) + 1;

struct Spec16Smem {
  double2 tw[kN16];
  // transpose [line][n2][k1] (row stride 17: conflict-free both ways),
  // reused as natural-order lines [line][pad(k)]
  union {
    double2 t[kL16][kR][kR + 1];
    double2 nat[kL16 * kLP16];
  };
  ZLinesT<2 * kL16> zl;
};

__device__ __forceinline__ double2 *nat16(Spec16Smem &sm, int line) {
  return sm.nat + line * kLP16;
}

template <bool kInv>
__device__ __forceinline__ void fft4(double2 &a0, double2 &a1, double2 &a2,
                                     double2 &a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  const double2 s13 = cadd(a1, a3), d13 = csub(a1, a3);
  // forward: -i d13; inverse: +i d13
  const double2 jd = kInv ? make_double2(-d13.y, d13.x)
                          : make_double2(d13.y, -d13.x);
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, jd);
  a3 = csub(d02, jd);
}

// exp(-+ 2 pi i p / 16), p = j1 m2 in 0 .. 9
template <bool kInv>
__device__ __forceinline__ double2 w16(int p) {
  constexpr double c1 = 0.92387953251128673848, s1 = 0.38268343236508978178;
  constexpr double h = 0.70710678118654752440;
  const double cs[10] = {1.0, c1, h, s1, 0.0, -s1, -h, -c1, -1.0, -c1};
  const double sn[10] = {0.0, s1, h, c1, 1.0, c1, h, s1, 0.0, -s1};
  return make_double2(cs[p], kInv ? sn[p] : -sn[p]);
}

// 16-point DFT in registers; X[k] ends in v[4 (k & 3) + (k >> 2)]
template <bool kInv>
__device__ __forceinline__ void fft16(double2 (&v)[kR]) {
#pragma unroll
  for (int m2 = 0; m2 < 4; ++m2) fft4<kInv>(v[m2], v[4 + m2], v[8 + m2], v[12 + m2]);
#pragma unroll
  for (int j1 = 1; j1 < 4; ++j1)
#pragma unroll
    for (int m2 = 1; m2 < 4; ++m2)
      v[4 * j1 + m2] = cmul(v[4 * j1 + m2], w16<kInv>(j1 * m2));
#pragma unroll
  for (int j1 = 0; j1 < 4; ++j1)
    fft4<kInv>(v[4 * j1], v[4 * j1 + 1], v[4 * j1 + 2], v[4 * j1 + 3]);
}
__device__ __forceinline__ int perm16(int k) { return 4 * (k & 3) + (k >> 2); }

// v (thread c's x[16 n1 + c]) -> u (X[c + 16 k2] at u[perm16(k2)]); the
// transpose buffer of `line` is free on entry and on exit
template <bool kInv>
__device__ __forceinline__ void fft256(Spec16Smem &sm, int line, int c,
                                       double2 (&v)[kR]) {
  fft16<kInv>(v);
#pragma unroll
  for (int k1 = 0; k1 < kR; ++k1) {
    double2 y = v[perm16(k1)];
    if (k1) {
      double2 w = sm.tw[(c * k1) & (kN16 - 1)];  // shared: no __ldg
      if (kInv) w.y = -w.y;
      y = cmul(y, w);
    }
    sm.t[line][c][k1] = y;
  }
  __syncthreads();
#pragma unroll
  for (int n2 = 0; n2 < kR; ++n2) v[n2] = sm.t[line][n2][c];
  fft16<kInv>(v);
}

__device__ __forceinline__ void load_tw16(Spec16Smem &sm, const double2 *tw) {
  for (int t = threadIdx.x; t < kN16; t += blockDim.x) sm.tw[t] = tw[t];
}

// pass 1 for sz == 256 (same output as k_spec_fwd_z)
template <bool kSlab>
__global__ void __launch_bounds__(kT16)
    k_spec_fwd_z16(SpecPlan sp, const double *__restrict__ r,
                   const int *done) {
  SPEC_DONE_RETURN;
  __shared__ Spec16Smem sm;
  load_tw16(sm, sp.twz);
  const int line = threadIdx.x >> 4, c = threadIdx.x & (kR - 1);
  const int nk = sp.nkz;
  const int32_t npairs = sp.nxl * sp.sy / 2;
  const int32_t ntiles = (npairs + kL16 - 1) / kL16;
  for (int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t g0 = tile * kL16;
    zlines_fill(sp, 2 * g0, 2 * kL16, sm.zl);
    __syncthreads();
    double2 v[kR];
    const bool ok = g0 + line < npairs;
    const int32_t b0 = sm.zl.base[2 * line], b1 = sm.zl.base[2 * line + 1];
#pragma unroll
    for (int n1 = 0; n1 < kR; ++n1)
      v[n1] = ok ? make_double2(r[b0 + kR * n1 + c], r[b1 + kR * n1 + c])
                 : make_double2(0.0, 0.0);
    fft256<false>(sm, line, c, v);
    __syncthreads();  // every transpose read is done: reuse as natural order
    double2 *zb = nat16(sm, line);
#pragma unroll
    for (int k2 = 0; k2 < kR; ++k2) zb[pad(c + kR * k2)] = v[perm16(k2)];
    __syncthreads();
    {
      // thread: real line jj of the tile, wavenumbers kz0, kz0 + 8, ...
      const int jj = threadIdx.x & (2 * kL16 - 1), kz0 = threadIdx.x >> 4;
      const int j = jj >> 1, side = jj & 1;
      const int32_t lx = sm.zl.x[jj], ly = sm.zl.y[jj];
      double2 *dst = sp.s + (int64_t)ly * nk * sp.sx + lx;
      const double2 *f = nat16(sm, j);
      if (g0 + j < npairs) {
#pragma unroll 4
        for (int kz = kz0; kz < nk; kz += kT16 / (2 * kL16)) {
          const double2 zk = f[pad(kz)];
          const double2 zm = f[pad((kN16 - kz) & (kN16 - 1))];
          const double2 o =
              side == 0
                  ? make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y))
                  : make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
          if (kSlab)
            *spec_at(sp, lx, ly, kz) = o;
          else
            dst[(int64_t)kz * sp.sx] = o;
        }
      }
    }
    __syncthreads();
  }
}

// passes 2 / 4 for sx == 256: complex FFT along X, in place
template <bool kInv>
__global__ void __launch_bounds__(kT16)
    k_spec_x16(SpecPlan sp, const int *done) {
  SPEC_DONE_RETURN;
  __shared__ Spec16Smem sm;
  load_tw16(sm, sp.twx);
  const int line = threadIdx.x >> 4, c = threadIdx.x & (kR - 1);
  const int64_t nlines =
      (int64_t)sp.sy * (sp.kz0[sp.rank + 1] - sp.kz0[sp.rank]);
  const int64_t ntiles = (nlines + kL16 - 1) / kL16;
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t l = tile * kL16 + line;
    const bool ok = l < nlines;
    double2 *src = sp.s + l * kN16;
    double2 v[kR];
#pragma unroll
    for (int n1 = 0; n1 < kR; ++n1)
      v[n1] = ok ? __ldcg(src + kR * n1 + c) : make_double2(0.0, 0.0);
    fft256<kInv>(sm, line, c, v);
    if (ok) {
#pragma unroll
      for (int k2 = 0; k2 < kR; ++k2) src[c + kR * k2] = v[perm16(k2)];
    }
    __syncthreads();  // the transpose buffer is free for the next tile
  }
}

// pass 5 for sz == 256 (same output as k_spec_inv_z)
template <bool kSums, bool kSlab>
__global__ void __launch_bounds__(kT16, 4)
    k_spec_inv_z16(SpecPlan sp, const double *__restrict__ r,
                   double *__restrict__ z, CgFuse fz, const int *done) {
  SPEC_DONE_RETURN;
  __shared__ Spec16Smem sm;
  load_tw16(sm, sp.twz);
  const int line = threadIdx.x >> 4, c = threadIdx.x & (kR - 1);
  constexpr int half = kN16 / 2;
  const int32_t npairs = sp.nxl * sp.sy / 2;
  const int32_t ntiles = (npairs + kL16 - 1) / kL16;
  double sums[3] = {0.0, 0.0, 0.0};
  for (int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t g0 = tile * kL16;
    zlines_fill(sp, 2 * g0, 2 * kL16, sm.zl);
    __syncthreads();
    // Hermitian extension of the two real lines' spectra, loaded with the
    // lines of the tile adjacent (coalesced), into natural order
    {
      // thread: line pair j of the tile, wavenumbers k0, k0 + 16, ...; the
      // loads of a half are issued back to back (lines are clamped, so
      // every address is valid).  Slab plans: the inverse transpose, loads
      // from the kz owner.
      const int j = threadIdx.x & (kL16 - 1), k0 = threadIdx.x >> 3;
      constexpr int kStep = kT16 / kL16, kH = kN16 / kStep / 2;
      const bool okj = g0 + j < npairs;
      const int32_t xa = sm.zl.x[2 * j], ya = sm.zl.y[2 * j];
      const int32_t xb = sm.zl.x[2 * j + 1], yb = sm.zl.y[2 * j + 1];
      const double2 *pa = sp.s + (int64_t)ya * sp.nkz * sp.sx + xa;
      const double2 *pb = sp.s + (int64_t)yb * sp.nkz * sp.sx + xb;
      double2 *dst = nat16(sm, j);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        double2 av[kH], bv[kH];
#pragma unroll
        for (int i = 0; i < kH; ++i) {
          const int k = k0 + kStep * (hh * kH + i);
          const int kk = k <= half ? k : kN16 - k;
          av[i] = __ldcg(kSlab ? spec_at(sp, xa, ya, kk)
                               : pa + (int64_t)kk * sp.sx);
          bv[i] = __ldcg(kSlab ? spec_at(sp, xb, yb, kk)
                               : pb + (int64_t)kk * sp.sx);
        }
#pragma unroll
        for (int i = 0; i < kH; ++i) {
          const int k = k0 + kStep * (hh * kH + i);
          const double2 a = av[i], b = bv[i];
          double2 v = k <= half ? make_double2(a.x - b.y, a.y + b.x)
                                : make_double2(a.x + b.y, b.x - a.y);
          if (!okj) v = make_double2(0.0, 0.0);
          dst[pad(k)] = v;
        }
      }
    }
    __syncthreads();
    double2 v[kR];
    const double2 *zb = nat16(sm, line);
#pragma unroll
    for (int n1 = 0; n1 < kR; ++n1) v[n1] = zb[pad(kR * n1 + c)];
    __syncthreads();  // natural-order reads done: the buffer is the transpose
    fft256<true>(sm, line, c, v);
    if (g0 + line < npairs) {
      const int32_t b0 = sm.zl.base[2 * line], b1 = sm.zl.base[2 * line + 1];
#pragma unroll
      for (int k2 = 0; k2 < kR; ++k2) {
        const double2 o = v[perm16(k2)];
        const int32_t i0 = b0 + c + kR * k2, i1 = b1 + c + kR * k2;
        z[i0] = o.x;
        z[i1] = o.y;
        if (kSums) {
          const double r0 = r[i0], r1 = r[i1];
          sums[0] += o.x + o.y;
          sums[1] += r0 * o.x + r1 * o.y;
          sums[2] += r0 + r1;
        }
      }
    }
    __syncthreads();
  }
  if (kSums) {
    double tot[3];
    if (grid_reduce<3>(sums, fz.partials, fz.counter, tot))
      cg_fin_z(fz.st, tot[0], tot[1], tot[2], sp.sx * sp.sy * sp.sz,
               fz.initial != 0);
  }
}

// ---------------------------------------------------------------------------
// setup

__global__ void __launch_bounds__(kBlock) k_spec_tables(SpecPlan sp) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double s, c;
  if (t < sp.sx) {
    sincospi(2.0 * t / sp.sx, &s, &c);
    sp.twx[t] = make_double2(c, -s);
    sp.lx[t] = sp.sx > 1 ? 2.0 - 2.0 * c : 0.0;
  }
  if (t < sp.sz) {
    sincospi(2.0 * t / sp.sz, &s, &c);
    sp.twz[t] = make_double2(c, -s);
    if (t < sp.nkz) sp.lz[t] = 2.0 - 2.0 * c;
  }
}

// plane means of the level-0 face weights, one CTA per Y plane
__global__ void __launch_bounds__(kBlock)
    k_spec_planes(MgLevel L, SpecPlan sp, const int *done) {
  SPEC_DONE_RETURN;
  const int y = blockIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  const int64_t m = (int64_t)sp.nxl * L.sz;
  for (int64_t e = threadIdx.x; e < m; e += blockDim.x) {
    const int64_t x = e / L.sz + sp.xoff, zz = e - (x - sp.xoff) * L.sz;
    const int64_t i = (x * L.sy + y) * L.sz + zz;
    v[0] += L.wx[i];
    v[1] += L.wy[i];
    v[2] += L.wz[i];
  }
  block_reduce<3>(v);
  if (threadIdx.x == 0) {
    sp.ax[y] = v[0];
    sp.ay[y] = v[1];
    sp.az[y] = v[2];
  }
}

// plane sums (over all ranks) -> plane means
__global__ void __launch_bounds__(kBlock) k_spec_plane_mean(SpecPlan sp) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 3 * sp.sy) sp.ax[t] /= (double)sp.sx * sp.sz;
}

// ---------------------------------------------------------------------------
// host side

static bool pow2_in(int n, int lo, int hi) {
  return n >= lo && n <= hi && (n & (n - 1)) == 0;
}

// PF_SPEC_GENERIC=1: the Stockham kernels for every length (comparison)
static const bool g_spec_generic = [] {
  const char *e = getenv("PF_SPEC_GENERIC");
  return e && e[0] == '1';
}();

bool spec_ok(int dim, int sx, int sy, int sz, int px, int pz) {
  if (!pz || !pow2_in(sz, 4, kFftElems) || sy < 2) return false;
  if (dim == 3) return px && pow2_in(sx, 2, kFftElems);
  return sx == 1 && sy % 2 == 0;
}

void spec_plan(SpecPlan &sp, int sx, int sy, int sz) {
  sp = SpecPlan{};
  sp.sx = sx;
  sp.sy = sy;
  sp.sz = sz;
  sp.nkz = sz / 2 + 1;
  sp.lpx = std::max(1, kFftElems / sx);
  sp.lpz = std::max(1, kFftElems / sz);
  sp.nxl = sx;
  sp.xoff = sp.x0 = sp.rank = 0;
  sp.world = 1;
  sp.kz0[0] = 0;
  sp.kz0[1] = sp.nkz;
}

void spec_slab_plan(SpecPlan &sp, int nxl, int x0, int rank, int world) {
  sp.nxl = nxl;
  sp.xoff = 1;
  sp.x0 = x0;
  sp.rank = rank;
  sp.world = world;
  const int base = sp.nkz / world, rem = sp.nkz % world;
  sp.kz0[0] = 0;
  for (int q = 0; q < world; ++q)
    sp.kz0[q + 1] = sp.kz0[q] + base + (q < rem ? 1 : 0);
}

static int nkz_max(const SpecPlan &sp) {
  int m = 0;
  for (int q = 0; q < sp.world; ++q)
    m = std::max(m, sp.kz0[q + 1] - sp.kz0[q]);
  return m;
}

static bool spec_is_slab(const SpecPlan &sp) { return sp.xoff != 0; }

static int64_t al(int64_t b) { return (b + 255) / 256 * 256; }

int64_t spec_slab_bytes(const SpecPlan &sp) {
  return al((int64_t)sp.sy * nkz_max(sp) * sp.sx * 16);
}

void spec_slab_bind(SpecPlan &sp, const CommHost &c) {
  for (int q = 0; q < sp.world; ++q)
    sp.peer_s[q] = reinterpret_cast<double2 *>(c.host.peer[q] + c.spec_off);
  sp.s = sp.peer_s[sp.rank];
}

int64_t spec_bytes(const SpecPlan &sp) {
  // the work array of a slab plan lives in the comm's symmetric buffer
  const int64_t ns = (int64_t)sp.sy * nkz_max(sp) * sp.sx;
  return (spec_is_slab(sp) ? 0 : al(ns * 16)) + 2 * al(ns * 8) +
         al(3 * sp.sy * 8) + al(sp.sx * 16) + al(sp.sz * 16) +
         al(sp.sx * 8) + al(sp.nkz * 8);
}

char *spec_bind(SpecPlan &sp, char *q) {
  const int64_t ns = (int64_t)sp.sy * nkz_max(sp) * sp.sx;
  if (!spec_is_slab(sp)) {
    sp.s = reinterpret_cast<double2 *>(q);
    sp.peer_s[0] = sp.s;
    q += al(ns * 16);
  }
  sp.cw = reinterpret_cast<double *>(q);
  q += al(ns * 8);
  sp.iw = reinterpret_cast<double *>(q);
  q += al(ns * 8);
  sp.ax = reinterpret_cast<double *>(q);
  sp.ay = sp.ax + sp.sy;
  sp.az = sp.ax + 2 * sp.sy;
  q += al(3 * sp.sy * 8);
  sp.twx = reinterpret_cast<double2 *>(q);
  q += al(sp.sx * 16);
  sp.twz = reinterpret_cast<double2 *>(q);
  q += al(sp.sz * 16);
  sp.lx = reinterpret_cast<double *>(q);
  q += al(sp.sx * 8);
  sp.lz = reinterpret_cast<double *>(q);
  q += al(sp.nkz * 8);
  return q;
}

template <typename... KArgs, typename... Args>
static void launch_smem(void (*kernel)(KArgs...), int grid, int block,
                        size_t smem, cudaStream_t stream, Args... args) {
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  count_launch();
  kernel<<<grid, block, smem, stream>>>(args...);
}

int spec_setup(const MgLevel &l0, const SpecPlan &sp, cudaStream_t s,
               const int *done, const Plan *pl) {
  if (spec_is_slab(sp) && (!pl || !pl->comm)) {
    set_error("spectral preconditioner of a slab plan: no communicator "
              "attached (pf_plan_attach_comm)");
    return PF_ERR_ARG;
  }
  launch(k_spec_tables, grid_for(std::max(sp.sx, sp.sz)), kBlock, s, sp);
  launch(k_spec_planes, sp.sy, kBlock, s, l0, sp, done);
  if (pl) {
    int rc = comm_vec_allreduce(*pl, sp.ax, 3 * sp.sy, 0, s);
    if (rc) return rc;
  }
  launch(k_spec_plane_mean, grid_for(3 * sp.sy), kBlock, s, sp);
  {
    const int64_t ncol =
        (int64_t)(sp.kz0[sp.rank + 1] - sp.kz0[sp.rank]) * sp.sx;
    launch_smem(k_spec_factors, grid_for(ncol, kYThreads), kYThreads,
                3 * sizeof(double) * sp.sy, s, sp, done);
  }
  PF_LAUNCH_CHECK("spec_setup");
  return PF_OK;
}


int spec_apply(const MgLevel &l0, const SpecPlan &sp, const double *r,
               double *z, cudaStream_t s, const int *done, cudaEvent_t *ev,
               const CgFuse *fuse, int red_blocks, const Plan *pl) {
  (void)l0;
  if (spec_is_slab(sp) && (!pl || !pl->comm)) {
    set_error("spectral preconditioner of a slab plan: no communicator");
    return PF_ERR_ARG;
  }
  // slab plans: the forward Z pass stores into the kz owners' spectra and
  // the inverse Z pass loads from them; barriers separate the all-to-all
  // from the owner-local X / Y passes (no-ops on a single GPU)
  auto barrier = [&]() {
    if (pl) comm_barrier(*pl, s);
  };
  auto mark = [&](int k) {
    if (ev) cudaEventRecord(ev[k], s);
  };
  const int64_t npairs = (int64_t)sp.nxl * sp.sy / 2;
  const int zt = (int)std::min<int64_t>((npairs + sp.lpz - 1) / sp.lpz,
                                        1 << 20);
  const size_t zsm = 2 * sizeof(double2) * sp.lpz * padded_len(sp.sz);
  const int nkl = sp.kz0[sp.rank + 1] - sp.kz0[sp.rank];
  const int64_t xlines = (int64_t)sp.sy * nkl;
  const int xt = (int)std::min<int64_t>((xlines + sp.lpx - 1) / sp.lpx,
                                        1 << 20);
  const size_t xsm = 2 * sizeof(double2) * sp.lpx * padded_len(sp.sx);
  const int64_t ncol2 = 2 * (int64_t)nkl * sp.sx;
  mark(0);
  const bool z16 = sp.sz == kN16 && !g_spec_generic;
  const bool x16 = sp.sx == kN16 && !g_spec_generic;
  const int zt16 = (int)std::min<int64_t>((npairs + kL16 - 1) / kL16, 1 << 20);
  const int xt16 = (int)std::min<int64_t>((xlines + kL16 - 1) / kL16, 1 << 20);
  const bool slab = sp.world > 1;
  if (z16 && slab)
    launch(k_spec_fwd_z16<true>, zt16, kT16, s, sp, r, done);
  else if (z16)
    launch(k_spec_fwd_z16<false>, zt16, kT16, s, sp, r, done);
  else
    launch_smem(k_spec_fwd_z, zt, kFftThreads, zsm, s, sp, r, done);
  barrier();
  mark(1);
  if (x16)
    launch(k_spec_x16<false>, xt16, kT16, s, sp, done);
  else if (sp.sx > 1)
    launch_smem(k_spec_x<false>, xt, kFftThreads, xsm, s, sp, done);
  mark(2);
  launch_smem(k_spec_ysolve, grid_for(ncol2, kYThreads), kYThreads,
              3 * sizeof(double) * sp.sy, s, sp, done);
  mark(3);
  if (x16)
    launch(k_spec_x16<true>, xt16, kT16, s, sp, done);
  else if (sp.sx > 1)
    launch_smem(k_spec_x<true>, xt, kFftThreads, xsm, s, sp, done);
  barrier();
  mark(4);
  if (fuse && fuse->st) {
    // the fused z-sums end in a cross-rank allreduce, which no rank leaves
    // before every rank's loads are done: it doubles as the closing barrier
    if (z16)
      launch(slab ? k_spec_inv_z16<true, true> : k_spec_inv_z16<true, false>,
             std::min(zt16, red_blocks), kT16, s, sp, r, z, *fuse, done);
    else
      launch_smem(k_spec_inv_z<true>, std::min(zt, red_blocks), kFftThreads,
                  zsm, s, sp, r, z, *fuse, done);
  } else {
    if (z16)
      launch(slab ? k_spec_inv_z16<false, true> : k_spec_inv_z16<false, false>,
             zt16, kT16, s, sp, r, z, CgFuse{nullptr, nullptr, nullptr, 0},
             done);
    else
      launch_smem(k_spec_inv_z<false>, zt, kFftThreads, zsm, s, sp, r, z,
                  CgFuse{nullptr, nullptr, nullptr, 0}, done);
    if (!(fuse && fuse->caller_closes)) barrier();
  }
  mark(5);
  PF_LAUNCH_CHECK("spec_apply");
  return PF_OK;
}

}  // namespace pf
