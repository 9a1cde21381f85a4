// bicg_nm.cuh -- BiCGStab passes with the two-sweep Jacobi (Neumann-2)
// polynomial right preconditioner, fused into one 2.5D-tiled sweep each.
// Included by solvers.cu inside namespace pf (uses TileGeo, wrap, cp_async8).
//
// The reference preconditions its momentum BiCGStab with ILU(0)
// (S/linalg.py:98-108, S/_kernels_c.pyx:66-149), a sequential triangular
// solve.  Here the preconditioner is two Jacobi sweeps,
//     M^-1 = D^-1 (2 I - A D^-1) = D^-1 - D^-1 N D^-1     (A = D + N),
// so that   A M^-1 y = y - N D^-1 N D^-1 y.
// On the C4 momentum operators it halves the Jacobi iteration count
// (forward 6 -> 3, adjoint 9 -> 5 lock-step iterations; the reference's
// ILU(0) takes 2 forward).  Both stencil applications of a pass run on chip:
// a CTA owns an 8 x 32 (Y, Z) column tile and marches along X; per plane q
//   convert  g1 = D^-1 y  of plane q on the tile + 2-cell halo (from the raw
//            inputs r, p, v, 1/A_jj staged by cp.async one plane ahead),
//   stage 1  q1 = D^-1 (N g1)  of plane q-1 on the tile + 1-cell halo,
//   stage 2  out = y - N q1    of plane q-2 on the tile,
// so every input array is read from HBM once per cell (the halos and the
// four chunk-boundary planes come mostly from L2) and no intermediate
// leaves the SM.  Only the six off-diagonal rows of A are read (N); the
// diagonal enters through 1/A_jj.  Two barriers per plane step.
//
// The iterate is kept in preconditioned form: x = x0 + M^-1 z, and one
// closing pass forms x once per solve.  The x/r update of iteration k is
// folded into the pv pass of iteration k+1 (MODE 3): that pass forms
// s = r - alpha v, r' = s - omega t and p' = r' + beta (p - omega v) at
// every stencil point from r, v, p, t, stores r' and z += alpha p + omega s
// at its own cells, and applies A M^-1 to p'.  beta needs r^.r' before the
// pass: the st pass sums r^.s and r^.t too, and r^.r' = r^.s - omega r^.t
// (linearity; S/linalg.py:206-209 forms the same dot directly).  Per
// iteration the passes move 296 + 152 B/cell instead of 200 + 128 + 192.
//
// Slab plans (one ghost plane per side): stage 1 at a ghost plane would
// need the raw inputs two planes outside the slab.  Instead each pass first
// runs in edge mode (`qedge`): stage 1 only, on the first and last owned
// planes, stored to Q; the halo exchange moves those planes into the
// neighbours' ghost planes of Q, and the main pass (`qghost` = Q) reads its
// stage-1 value at a ghost plane from there.  Stage 2 needs a ghost plane's
// q1 only at its own column (the X neighbour), so one plane of Q suffices.

//
// Addressing: every in-plane offset is computed once per tile, per plane
// only the wrapped X plane base changes; all array pointers (per component,
// per stencil row) arrive pre-offset in the kernel parameters (NmArgs), so
// a global address is one add on a constant-bank operand; shared-memory
// ring slots are rotating base registers; the raw inputs move as 16-byte
// pairs along Z (the 36-wide halo row and the tile origin are even, and a
// pair never straddles a periodic seam or a wall).  The plane loop is
// peeled (prologue planes convert only / convert + stage 1) and the common
// case of all three components active is its own instantiation, so the
// steady-state step carries no per-component or per-stage tests.

constexpr int kNY = kTY + 4, kNZ = kTZ + 4;           // tile + 2-cell halo
constexpr int kNP = kNY * kNZ;                         // 432 cells per plane
constexpr int kNPairs = kNP / 2;                       // 216 Z-pairs
constexpr int kNRing1 = (kTY + 2) * (kTZ + 2) - kTY * kTZ;  // 84 halo-1 cells
constexpr int kNZ1 = kTZ + 2;                          // q1 row (halo 1)
constexpr int kNP1 = (kTY + 2) * kNZ1;                 // 340 q1 cells
static_assert(kNZ % 2 == 0 && kNPairs <= kTileThreads, "pair layout");

// shared memory, in doubles: raw[13][kNP] (r, v, p, t x 3, 1/A) |
// g1[3 slots][3][kNP] | q1[4 slots][3][kNP1] | iteration scalars [3][3]
// (q1 lives on the tile + 1-cell halo only, 340 cells per plane: measured
// C4 x/r + pv pass 1114 -> 937 us against the 432-cell layout.  A
// three-slot q1 ring and per-pass raw buffers (100.6 / 90.2 / 79.8 KB)
// were measured 1 % slower again.)
// (q1 keeps four planes: stage 2 of plane q-3 reads q-4, q-3, q-2 while
// stage 1 writes q-1, and reads its X neighbours from the ring)
constexpr int kNmRawN = 13, kNmDi = 12;  // raw arrays; 1/A's slot
constexpr int kNmRaw = 0, kNmG1 = kNmRawN * kNP, kNmQ1 = kNmG1 + 9 * kNP,
              kNmCo = kNmQ1 + 12 * kNP1, kNmCf = kNmCo + 10,
              kNmEnd = kNmCf + 12 * kTileThreads;
// The transposed passes park each plane's own (gathered) row for its stage 2
// two plane steps later (two slots x 6 rows x 256 cells): adjoint st 763 ->
// 739 us; the forward passes, whose own row is one coalesced load per face,
// measured 1.7 % slower with it and keep the smaller buffer (more L1)
template <bool kTrans>
constexpr size_t nm_smem() {
  return sizeof(double) * (kTrans ? kNmEnd : kNmCf);  // 133,328 / 108,752 B
}

// halo-1 ring cell k (0..83) in plane coordinates
__device__ __forceinline__ void nm_ring1(int k, int &sy, int &sz) {
  if (k < 2 * (kTZ + 2)) {
    sy = k < kTZ + 2 ? 1 : kTY + 2;
    sz = 1 + k % (kTZ + 2);
  } else {
    const int k2 = k - 2 * (kTZ + 2);
    sy = 2 + (k2 >> 1);
    sz = (k2 & 1) ? kTZ + 2 : 1;
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
               "l"(gmem)
               : "memory");
}

// Pointers of one pass, pre-offset on the host (the kernel adds cell
// indices only).  row[f]: stencil row of face f (-x +x -y +y -z +z) of A,
// or for A^T the neighbour's back-face row, read at the neighbour.
struct NmArgs {
  const double *src[4][3];  // raw array k of component q: r, v, p, t | z
  double *rout[3];          // MODE 3: r' (the other r buffer)
  double *zio[3];           // MODE 3: the preconditioned iterate z
  const double *dinv;
  const double *row[6];
  const double *rhat[3];
  double *out1[3];          // pv: p'   | close: x   | edge: Q
  double *out2[3];          // pv: v'   | st: t
  const double *qghost[3];  // slab ghost-plane stage 1 (null: none)
  int32_t X, Y, Z, px, py, pz;
  int32_t sX;               // cells per X plane
};

// in-plane addressing of one stencil row (own or halo-1 cell): its offset
// in the plane and, for the transposed gathers, its Y/Z neighbours' (-1
// outside a walled box)
struct NmRow {
  int32_t off, ym, yp, zm, zp;
  bool ok;  // inside the box (Y, Z)
};

__device__ __forceinline__ NmRow nm_row(const NmArgs &g, int32_t gy0,
                                        int32_t gz0) {
  NmRow r;
  bool oy, oz, o;
  const int32_t y = wrap(gy0, g.Y, g.py, oy);
  const int32_t z = wrap(gz0, g.Z, g.pz, oz);
  r.ok = oy && oz;
  r.off = y * g.Z + z;
  int32_t c = wrap(y - 1, g.Y, g.py, o);
  r.ym = o ? c * g.Z + z : -1;
  c = wrap(y + 1, g.Y, g.py, o);
  r.yp = o ? c * g.Z + z : -1;
  c = wrap(z - 1, g.Z, g.pz, o);
  r.zm = o ? y * g.Z + c : -1;
  c = wrap(z + 1, g.Z, g.pz, o);
  r.zp = o ? y * g.Z + c : -1;
  return r;
}

// plane base (first cell) of plane x, -1 outside a walled box
__device__ __forceinline__ int32_t nm_pbase(const NmArgs &g, int32_t x) {
  if (x < 0) return g.px ? (x + g.X) * g.sX : -1;
  if (x >= g.X) return g.px ? (x - g.X) * g.sX : -1;
  return x * g.sX;
}

// the six off-diagonal coefficients of a row at plane base b (kTrans: the
// X neighbours' rows at plane bases bm / bp); zero across walls
template <bool kTrans>
__device__ __forceinline__ void nm_coefs(const NmArgs &g, int32_t b,
                                         int32_t bm, int32_t bp,
                                         const NmRow &rw, double (&cf)[6]) {
  if (!kTrans) {
    const int32_t i = b + rw.off;
#pragma unroll
    for (int f = 0; f < 6; ++f) cf[f] = __ldg(g.row[f] + i);
    return;
  }
  cf[0] = bm >= 0 ? __ldg(g.row[0] + bm + rw.off) : 0.0;
  cf[1] = bp >= 0 ? __ldg(g.row[1] + bp + rw.off) : 0.0;
  cf[2] = rw.ym >= 0 ? __ldg(g.row[2] + b + rw.ym) : 0.0;
  cf[3] = rw.yp >= 0 ? __ldg(g.row[3] + b + rw.yp) : 0.0;
  cf[4] = rw.zm >= 0 ? __ldg(g.row[4] + b + rw.zm) : 0.0;
  cf[5] = rw.zp >= 0 ? __ldg(g.row[5] + b + rw.zp) : 0.0;
}

// MODE 0 (pass pv): y = p' = r + beta (p - omega v) (kFirst: p' = r);
//                   outputs p', v' = A M^-1 p'; sums r^.v' -> alpha
// MODE 1 (pass st): y = s = r - alpha v'; outputs t = A M^-1 s; sums s.s,
//                   t.t, t.s -> early exit / omega
// MODE 2 (close):   y = z (the preconditioned iterate); x += M^-1 z
//                   (stage 1 only, no reduction)
// MODE 3 (x/r + pv): iteration k's update fused into iteration k+1's pv
//                   (above): r', z and p', v' = A M^-1 p'; sums r^.v',
//                   |r'|^2 -> convergence, alpha
// edge (MODE 0 / 1): stage 1 only on one plane per chunk, stored to Q
template <bool kTrans, int MODE, bool kFirst = false, int kMinB = 2>
__global__ void __launch_bounds__(kTileThreads, kMinB)
    k_bi_nm(const __grid_constant__ TileGeo tg,
            const __grid_constant__ NmArgs g, SolverState *st, double *partials,
            unsigned *counter, int edge) {
  if (MODE != 2 && st->all_done) return;
  constexpr int K = MODE == 1 ? 15 : MODE == 3 ? 6 : 3;
  constexpr bool kClose = MODE == 2;
  constexpr bool kRpv = MODE == 3;
  // arrays per component in the raw buffer: r, v, p (pv) | r, v (st) | z |
  // r, v, p, t (x/r + pv)
  constexpr int kArr = kClose || (MODE == 0 && kFirst) ? 1
                       : MODE == 0 ? 3 : MODE == 3 ? 4 : 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *const sm = reinterpret_cast<double *>(smem_raw);
  const int nc = st->ncomp;
  bool act[3], pend[3], appl[3];
  // the iteration scalars live in shared memory (read where y is formed):
  // pv: beta, omega | st: alpha | x/r + pv: alpha, omega, beta
  double *const c0 = sm + kNmCo, *const c1 = sm + kNmCo + 3,
               *const c2 = sm + kNmCo + 6;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    // closing pass: the components that iterated and did not break down
    // (a breakdown restarts from zero unpreconditioned anyway)
    act[q] = q < nc && (kClose ? (st->c[q].active && !st->c[q].zero_rhs &&
                                  st->c[q].iter > 0 && !st->c[q].fail)
                               : !st->c[q].done);
    // x/r + pv: components that converged at s only take z += alpha p
    // ... unless the light pass (k_nm_xr) behind the last poll made it
    appl[q] = kRpv && q < nc && st->c[q].xr_applied;
    pend[q] = kRpv && q < nc && st->c[q].pending && !appl[q];
  }
  if (threadIdx.x < 3) {
    const int q = threadIdx.x;
    const bool ok = q < nc;
    c0[q] = !ok ? 0.0 : MODE == 0 ? st->c[q].beta : st->c[q].alpha;
    c1[q] = ok && (MODE == 0 || kRpv) ? st->c[q].omega : 0.0;
    c2[q] = ok && kRpv ? st->c[q].beta : 0.0;
  }
  const bool one = kClose || edge;
  const int tid = threadIdx.x;
  const int tz = tid % kTZ, ty = tid / kTZ;
  const int eo = (ty + 2) * kNZ + tz + 2;  // own cell's plane element
  const int eo1 = (ty + 1) * kNZ1 + tz + 1;  // ... in the q1 layout
  // the Z-pair this thread loads and converts, the halo-1 cell it smooths
  const bool has_pair = tid < kNPairs;
  const int psy = tid / (kNZ / 2), psz = 2 * (tid % (kNZ / 2));
  const int ep = psy * kNZ + psz;
  const bool has_r1 = tid < kNRing1;
  int r1y = 0, r1z = 0;
  if (has_r1) nm_ring1(tid, r1y, r1z);
  const int er = r1y * kNZ + r1z;
  const int er1 = (r1y - 1) * kNZ1 + r1z - 1;

  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;

  // the whole tile loop, specialised for "all three components active"
  auto run = [&](auto all_t) {
    constexpr bool kAll = decltype(all_t)::value;
    auto on = [&](int c) { return kAll || act[c]; };
    for (int tile = blockIdx.x; tile < tg.ntiles; tile += gridDim.x) {
      const int tzt = tile % tg.tz_tiles;
      const int rest = tile / tg.tz_tiles;
      const int tyt = rest % tg.ty_tiles;
      const int ch = rest / tg.ty_tiles;
      const int32_t y0 = tyt * kTY - 2, z0 = tzt * kTZ - 2;  // plane origin
      const int32_t xs = tg.x0 + ch * tg.xc;
      const int32_t xe = edge ? xs + 1 : min(xs + tg.xc, tg.x1);
      // in-plane addressing, fixed for the tile
      const NmRow own = nm_row(g, y0 + ty + 2, z0 + tz + 2);
      const NmRow ring = nm_row(g, y0 + r1y, z0 + r1z);
      bool okp;
      int32_t offp;
      {
        bool oy, oz;
        const int32_t gy = wrap(y0 + psy, g.Y, g.py, oy);
        const int32_t gz = wrap(z0 + psz, g.Z, g.pz, oz);
        okp = has_pair && oy && oz;
        offp = gy * g.Z + gz;
      }
      // raw inputs of plane x: one 16-byte copy per array of the pair;
      // zeros outside the box
      auto issue_plane = [&](int32_t x) {
        if (has_pair) {
          const int32_t b = nm_pbase(g, x);
          double *dst = sm + kNmRaw + ep;
          if (b < 0 || !okp) {
#pragma unroll
            for (int k = 0; k < kNmRawN; ++k)
              *reinterpret_cast<double2 *>(dst + k * kNP) =
                  make_double2(0.0, 0.0);
          } else {
            const int32_t j = b + offp;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              if (!on(q) && !pend[q]) continue;
#pragma unroll
              for (int k = 0; k < kArr; ++k)
                cp_async16(dst + (3 * k + q) * kNP, g.src[k][q] + j);
            }
            cp_async16(dst + kNmDi * kNP, g.dinv + j);
          }
        }
        cp_async_commit();
      };
      // y of element e of the raw buffer
      auto yval = [&](int e, int q) {
        const double *rw = sm + kNmRaw + e;
        const double rr = rw[q * kNP];
        if (kArr == 1) return rr;
        const double vv = rw[(3 + q) * kNP];
        if (kRpv) {
          const double om = c1[q];
          const double rn = (rr - c0[q] * vv) - om * rw[(9 + q) * kNP];
          return rn + c2[q] * (rw[(6 + q) * kNP] - om * vv);
        }
        return MODE == 0 ? rr + c0[q] * (rw[(6 + q) * kNP] - c1[q] * vv)
                         : rr - c0[q] * vv;
      };

      // ring slots: g1 of planes q-3 / q-2 / q-1 and q1 of planes q-5 /
      // q-4 / q-3 / q-2 at the start of step q; rotated every step
      int g1a = kNmG1, g1b = g1a + 3 * kNP, g1c = g1b + 3 * kNP;
      int q1a = kNmQ1, q1b = q1a + 3 * kNP1, q1c = q1b + 3 * kNP1,
          q1d = q1c + 3 * kNP1;
      // own-cell y of planes q-3, q-2, q-1, q
      double ya[3] = {0, 0, 0}, yb[3] = {0, 0, 0}, yc[3] = {0, 0, 0},
             yd[3] = {0, 0, 0};

      // stage-1-only passes (close, edge) smooth planes [xs, xe); the full
      // passes [xs - 1, xe], except a slab's ghost planes, whose q1 comes
      // from qghost (so the planes beyond them are never converted)
      const bool lo_g = g.qghost[0] && xs == tg.x0;
      const bool hi_g = g.qghost[0] && xe == tg.x1;
      const int32_t qbeg = one || lo_g ? xs - 1 : xs - 2;
      const int32_t qconv = one || hi_g ? xe : xe + 1;  // last converted

      // One plane step q:
      //   phase A (after B_a): convert plane q (g1, own y) and stage 2 of
      //     plane q-3 (out = y - N q1) -- independent work, interleaved;
      //   phase B (after B_b): stage 1 of plane q-1 (q1 = D^-1 N g1).
      // S1 / S2 select the stages (peeled prologue and epilogue steps).
      auto step = [&](int32_t q, auto s1_t, auto s2_t) {
        constexpr bool S1 = decltype(s1_t)::value;
        constexpr bool S2 = decltype(s2_t)::value;
        const int32_t x1 = q - 1, x3 = q - 3;
        const bool ghost1 = S1 && ((lo_g && x1 == xs - 1) ||
                                   (hi_g && x1 == xe));
        const int g1q = g1a;  // plane q goes to the oldest g1 slot
        // plane x1's N rows and 1/A (own, halo-1), x3's N rows and r^:
        // plain loads consumed after the barriers
        double cB[6], cR[6], cA[6];
        double djo = 0.0, djr = 0.0;
        int32_t b1 = -1;
        if (S1 && !ghost1) {
          b1 = nm_pbase(g, x1);
          if (b1 >= 0) {
            const int32_t bm = kTrans ? nm_pbase(g, x1 - 1) : 0;
            const int32_t bp = kTrans ? nm_pbase(g, x1 + 1) : 0;
            nm_coefs<kTrans>(g, b1, bm, bp, own, cB);
            djo = __ldg(g.dinv + b1 + own.off);
            if (!one && has_r1 && ring.ok) {
              nm_coefs<kTrans>(g, b1, bm, bp, ring, cR);
              djr = __ldg(g.dinv + b1 + ring.off);
            }
          }
        }
        double rh[3] = {0, 0, 0};
        int32_t i3 = 0;
        if (S2) {
          const int32_t b3 = nm_pbase(g, x3);
          i3 = b3 + own.off;
          if (!kTrans) nm_coefs<false>(g, b3, 0, 0, own, cA);
          {
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (on(c)) rh[c] = __ldg(g.rhat[c] + i3);
          }
        }
        // x/r + pv: the own cell's z of plane q, loaded ahead of the
        // barriers (its latency would otherwise sit inside phase A)
        double zq[3] = {0, 0, 0};
        int32_t iq = 0;
        if constexpr (kRpv) {
          if (!edge && q >= xs && q < xe) {
            iq = nm_pbase(g, q) + own.off;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if ((on(c) && !appl[c]) || pend[c]) zq[c] = g.zio[c][iq];
          }
        }
        if (ghost1) {
          // the neighbour rank's stage 1 of this plane (own column: only
          // stage 2's X neighbour reads it) into plane x1's q1 slot
          const int32_t ig = nm_pbase(g, x1) + own.off;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            sm[q1a + c * kNP1 + eo1] = on(c) ? __ldg(g.qghost[c] + ig) : 0.0;
        }
        cp_async_wait_all();
        __syncthreads();  // B_a: plane q's raw inputs have landed
        // phase A
        if (q <= qconv) {
          if (has_pair) {
            const double2 dj = *reinterpret_cast<const double2 *>(
                sm + kNmRaw + kNmDi * kNP + ep);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              if (!on(c)) continue;
              const double v0 = yval(ep, c), v1 = yval(ep + 1, c);
              *reinterpret_cast<double2 *>(sm + g1q + c * kNP + ep) =
                  make_double2(v0 * dj.x, v1 * dj.y);
            }
          }
          if (!one) {
#pragma unroll
            for (int c = 0; c < 3; ++c) yd[c] = on(c) ? yval(eo, c) : 0.0;
          }
          if constexpr (MODE == 0 && kFirst) if (!edge && q >= xs && q < xe) {
            // the first iteration starts the preconditioned iterate z at 0
            const int32_t io = nm_pbase(g, q) + own.off;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c < nc && g.zio[c]) g.zio[c][io] = 0.0;
          }
          if constexpr (kRpv) if (!edge && q >= xs && q < xe) {
            // iteration k's x/r update at the own cell of an owned plane
            const double *rw = sm + kNmRaw + eo;
            const int32_t io = iq;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              if (!on(c) && !pend[c]) continue;
              const double al = c0[c], pp = rw[(6 + c) * kNP];
              if (on(c)) {
                const double om = c1[c];
                const double sv = rw[c * kNP] - al * rw[(3 + c) * kNP];
                const double rn = sv - om * rw[(9 + c) * kNP];
                g.rout[c][io] = rn;
                if (!appl[c]) g.zio[c][io] = zq[c] + (al * pp + om * sv);
                acc[3 + c] += rn * rn;
              } else {
                g.zio[c][io] = zq[c] + al * pp;
              }
            }
          }
        }
        if (S2) {
          // the own row of plane x3: stage 1 loaded it two steps ago and
          // parked it in shared memory (own cell only, no barrier needed)
          if (kTrans) {
            const double *cf = sm + kNmCf + (x3 & 1) * 6 * kTileThreads + tid;
#pragma unroll
            for (int f = 0; f < 6; ++f) cA[f] = cf[f * kTileThreads];
          }
          // q1 of planes x3 - 1, x3, x3 + 1: slots q1b, q1c, q1d
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (!on(c)) continue;
            const double *qq = sm + q1c + c * kNP1 + eo1;
            const double off = cA[0] * sm[q1b + c * kNP1 + eo1] +
                               cA[1] * sm[q1d + c * kNP1 + eo1] +
                               cA[2] * qq[-kNZ1] + cA[3] * qq[kNZ1] +
                               cA[4] * qq[-1] + cA[5] * qq[1];
            const double out = ya[c] - off;
            g.out2[c][i3] = out;
            if constexpr (MODE == 0 || kRpv) {
              g.out1[c][i3] = ya[c];
              acc[c] += rh[c] * out;
            } else {
              acc[5 * c] += ya[c] * ya[c];
              acc[5 * c + 1] += out * out;
              acc[5 * c + 2] += out * ya[c];
              acc[5 * c + 3] += rh[c] * ya[c];   // r^.s
              acc[5 * c + 4] += rh[c] * out;     // r^.t
            }
          }
        }
        __syncthreads();  // B_b: g1(q) complete; the raw buffer is free
        if (q + 1 <= qconv) issue_plane(q + 1);
        else cp_async_commit();
        // phase B: stage 1 at x1 reads g1 of planes x1 - 1, x1, x1 + 1 =
        // slots g1b, g1c, g1q, writes q1 slot q1a
        if (S1 && !ghost1) {
          const double *gm = sm + g1b, *gc = sm + g1c, *gp = sm + g1q;
          const bool in1 = b1 >= 0;
          double *qn = sm + q1a;
          double qo[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            qo[c] = 0.0;
            if (!on(c) || !in1) continue;
            const int o = c * kNP + eo;
            qo[c] = djo * (cB[0] * gm[o] + cB[1] * gp[o] +
                           cB[2] * gc[o - kNZ] + cB[3] * gc[o + kNZ] +
                           cB[4] * gc[o - 1] + cB[5] * gc[o + 1]);
          }
          if (kTrans && !one && in1) {
            // stage 2 of plane x1 (two steps on) reuses this own row
            double *cf = sm + kNmCf + (x1 & 1) * 6 * kTileThreads + tid;
#pragma unroll
            for (int f = 0; f < 6; ++f) cf[f * kTileThreads] = cB[f];
          }
          if (kClose) {
            const int32_t i1 = b1 + own.off;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (on(c)) g.out1[c][i1] += gc[c * kNP + eo] - qo[c];
          } else if (one) {
            const int32_t i1 = b1 + own.off;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (on(c)) g.out1[c][i1] = qo[c];
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) qn[c * kNP1 + eo1] = qo[c];
            if (has_r1) {
              const bool okr = in1 && ring.ok;
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                if (!on(c)) continue;
                const int o = c * kNP + er;
                qn[c * kNP1 + er1] = okr ? djr * (cR[0] * gm[o] + cR[1] * gp[o] +
                                     cR[2] * gc[o - kNZ] +
                                     cR[3] * gc[o + kNZ] +
                                     cR[4] * gc[o - 1] + cR[5] * gc[o + 1])
                            : 0.0;
              }
            }
          }
        }
        // rotate: g1 (a,b,c) <- (b,c,q); q1 (a,b,c,d) <- (b,c,d,a) once
        // stage 1 wrote plane x1 into a; y (a,b,c,d) <- (b,c,d,-)
        g1a = g1b;
        g1b = g1c;
        g1c = g1q;
        if (S1) {
          const int t = q1a;
          q1a = q1b;
          q1b = q1c;
          q1c = q1d;
          q1d = t;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ya[c] = yb[c];
          yb[c] = yc[c];
          yc[c] = yd[c];
        }
      };

      __syncthreads();  // the previous tile is done with every buffer
      issue_plane(qbeg);
      using T = std::true_type;
      using F = std::false_type;
      int32_t q = qbeg;
      if (one) {
        // stage 1 on [xs, xe): convert xs - 1 and xs, then xs + 1 .. xe
        step(q++, F{}, F{});
        step(q++, F{}, F{});
        for (; q <= xe; ++q) step(q, T{}, F{});
      } else {
        // stage 1 of planes xs - 1 .. xe (steps xs .. xe + 1), stage 2 of
        // xs .. xe - 1 (steps xs + 3 .. xe + 2)
        for (; q < xs; ++q) step(q, F{}, F{});
        for (; q <= min(xs + 2, xe + 1); ++q) step(q, T{}, F{});
        for (; q <= xe + 1; ++q) step(q, T{}, T{});
        step(q, F{}, T{});
      }
      cp_async_wait_all();
    }
  };
  if (act[0] && act[1] && act[2])
    run(std::true_type{});
  else
    run(std::false_type{});
  (void)pend;

  if (kClose || edge) return;
  double tot[K];
  if (!grid_reduce<K>(acc, partials, counter, tot)) return;
  if constexpr (kRpv) {
    // iteration k completes: convergence on r', else iteration k + 1's
    // alpha (its rho is the st pass's rho_next, which beta used)
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      c.pending = 0;  // applied here or by the light pass
      c.xr_applied = 0;
      if (act[q]) {
        c.res = sqrt(tot[3 + q]);
        if (c.res <= c.tol_abs) {
          c.converged = 1;
          c.done = 1;
        } else if (c.iter >= c.maxiter) {
          c.done = 1;
        } else if (c.brk_next) {
          c.fail = 1;
          c.done = 1;
        } else {
          c.rho = c.rho_new;
          c.iter += 1;
          c.rho_new = c.rho_next;
          if (fabs(tot[q]) < DBL_MIN) {
            c.fail = 1;
            c.done = 1;
          } else {
            c.alpha = c.rho_new / tot[q];
          }
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
    return;
  }
  if constexpr (MODE == 0) {
    int all = 1;
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (act[q]) {
        if (fabs(tot[q]) < DBL_MIN) {
          c.fail = 1;
          c.done = 1;
        } else {
          c.alpha = c.rho_new / tot[q];
        }
      }
      if (!c.done) all = 0;
    }
    st->all_done = all;
  } else if constexpr (MODE == 1) {
    // all_done is left alone: the x/r + pv pass applies the early-exit
    // update; rho_next = r^.r' and beta for that pass
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (!act[q]) continue;
      c.res = sqrt(tot[5 * q]);
      if (c.res <= c.tol_abs) {
        c.converged = 1;
        c.done = 1;
        c.pending = 1;
      } else if (tot[5 * q + 1] < DBL_MIN) {
        c.fail = 1;
        c.done = 1;
      } else {
        c.omega = tot[5 * q + 2] / tot[5 * q + 1];
        c.rho_next = tot[5 * q + 3] - c.omega * tot[5 * q + 4];
        c.brk_next = fabs(c.rho_next) < DBL_MIN || fabs(c.omega) < DBL_MIN;
        c.beta = c.brk_next ? 0.0
                            : (c.rho_next / c.rho_new) * (c.alpha / c.omega);
      }
    }
  }
}
