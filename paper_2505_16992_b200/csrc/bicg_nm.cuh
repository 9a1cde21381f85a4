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
// The iterate is kept in preconditioned form: x = x0 + M^-1 z with
// z += alpha p + omega s (k_bi_xr<true>), and one closing pass (MODE 2)
// forms x once per solve.
//
// Slab plans (one ghost plane per side): stage 1 at a ghost plane would
// need the raw inputs two planes outside the slab.  Instead each pass first
// runs in edge mode (`qedge`): stage 1 only, on the first and last owned
// planes, stored to Q; the halo exchange moves those planes into the
// neighbours' ghost planes of Q, and the main pass (`qghost` = Q) reads its
// stage-1 value at a ghost plane from there.  Stage 2 needs a ghost plane's
// q1 only at its own column (the X neighbour), so one plane of Q suffices.

constexpr int kNY = kTY + 4, kNZ = kTZ + 4;           // tile + 2-cell halo
constexpr int kNRing2 = kNY * kNZ - kTY * kTZ;        // 176 halo-2 cells
constexpr int kNRing1 = (kTY + 2) * (kTZ + 2) - kTY * kTZ;  // 84 halo-1 cells
constexpr int kNRing2First = kTileThreads - kNRing2;  // threads 80.. convert
static_assert(kNRing1 <= kNRing2First + 4, "ring assignment");

struct NmSmem {
  double raw[10][kNY][kNZ];     // r x3, p x3 (pv) / v x3, v x3 (pv), 1/A
  double g1[3][3][kNY][kNZ];    // D^-1 y, planes q % 3
  double dv[2][kNY][kNZ];       // 1/A on the 1-halo, planes q % 2
  double q1[2][3][kNY][kNZ];    // D^-1 N g1, planes q % 2
};
constexpr size_t kNmSmem = sizeof(NmSmem);

// plane slot of a ring of three (planes run from -2)
__device__ __forceinline__ int mod3(int32_t x) { return (x + 3) % 3; }

// halo-2 ring cell k (0..175) of the (kNY, kNZ) plane
__device__ __forceinline__ void nm_ring2(int k, int &sy, int &sz) {
  if (k < 4 * kNZ) {
    const int row = k / kNZ;
    sy = row < 2 ? row : row + kTY;
    sz = k % kNZ;
  } else {
    const int k2 = k - 4 * kNZ, c = k2 & 3;
    sy = 2 + (k2 >> 2);
    sz = c < 2 ? c : c + kTZ;
  }
}
// halo-1 ring cell k (0..83)
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

// Off-diagonal coefficients of row (x, y, z) of A (kTrans: of A^T, gathered
// from the neighbours' back faces); zero across walls.  Faces: -x +x -y +y
// -z +z.
template <bool kTrans>
__device__ __forceinline__ void nm_coefs(const TileGeo &tg,
                                         const double *__restrict__ a,
                                         int64_t n, int32_t x, int32_t y,
                                         int32_t z, double (&cf)[6]) {
  const int64_t sX = (int64_t)tg.Y * tg.Z, sY = tg.Z;
  if (!kTrans) {
    const int64_t i = (int64_t)x * sX + (int64_t)y * sY + z;
#pragma unroll
    for (int f = 0; f < 6; ++f) cf[f] = __ldg(a + (int64_t)(1 + f) * n + i);
    return;
  }
  bool ok;
  int32_t c;
  c = wrap(x - 1, tg.X, tg.px, ok);
  cf[0] = ok ? __ldg(a + 2 * n + c * sX + (int64_t)y * sY + z) : 0.0;
  c = wrap(x + 1, tg.X, tg.px, ok);
  cf[1] = ok ? __ldg(a + 1 * n + c * sX + (int64_t)y * sY + z) : 0.0;
  c = wrap(y - 1, tg.Y, tg.py, ok);
  cf[2] = ok ? __ldg(a + 4 * n + x * sX + (int64_t)c * sY + z) : 0.0;
  c = wrap(y + 1, tg.Y, tg.py, ok);
  cf[3] = ok ? __ldg(a + 3 * n + x * sX + (int64_t)c * sY + z) : 0.0;
  c = wrap(z - 1, tg.Z, tg.pz, ok);
  cf[4] = ok ? __ldg(a + 6 * n + x * sX + (int64_t)y * sY + c) : 0.0;
  c = wrap(z + 1, tg.Z, tg.pz, ok);
  cf[5] = ok ? __ldg(a + 5 * n + x * sX + (int64_t)y * sY + c) : 0.0;
}

// MODE 0 (pass pv): y = p' = r + beta (p - omega v) (kFirst: p' = r);
//                   outputs p', v' = A M^-1 p'; sums r^.v' -> alpha
// MODE 1 (pass st): y = s = r - alpha v'; outputs t = A M^-1 s; sums s.s,
//                   t.t, t.s -> early exit / omega
// MODE 2 (close):   y = z (the preconditioned iterate); x += M^-1 z
//                   (stage 1 only, no reduction)
template <bool kTrans, int MODE, bool kFirst = false>
__global__ void __launch_bounds__(kTileThreads, 2)
    k_bi_nm(TileGeo tg, const double *__restrict__ a, BiVecs w, int par,
            int64_t n, SolverState *st, double *partials, unsigned *counter,
            const double *__restrict__ zin = nullptr,
            double *__restrict__ xout = nullptr,
            const double *__restrict__ qghost = nullptr,
            double *__restrict__ qedge = nullptr) {
  if (MODE != 2 && st->all_done) return;
  // edge mode: stage 1 of one plane per chunk, to qedge (no stage 2)
  const bool edge = qedge != nullptr;
  constexpr int K = MODE == 1 ? 9 : 3;
  constexpr bool kClose = MODE == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  NmSmem &sm = *reinterpret_cast<NmSmem *>(smem_raw);
  const int nc = st->ncomp;
  int act[3];
  double c0[3], c1[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    // closing pass: the components that iterated and did not break down
    // (a breakdown restarts from zero unpreconditioned anyway)
    act[q] = q < nc && (kClose ? (st->c[q].active && !st->c[q].zero_rhs &&
                                  st->c[q].iter > 0 && !st->c[q].fail)
                               : !st->c[q].done);
    c0[q] = q < nc ? (MODE == 0 ? st->c[q].beta : st->c[q].alpha) : 0.0;
    c1[q] = q < nc && MODE == 0 ? st->c[q].omega : 0.0;
  }
  const double *__restrict__ r = w.r;
  const double *__restrict__ dinv = w.dinv;
  const double *__restrict__ pin = w.p[par];
  const double *__restrict__ vin = MODE == 0 ? w.v[par] : w.v[par ^ 1];
  double *__restrict__ pout = w.p[par ^ 1];
  double *__restrict__ vout = MODE == 0 ? w.v[par ^ 1] : w.t;
  const int64_t sX = (int64_t)tg.Y * tg.Z, sY = tg.Z;
  const int tid = threadIdx.x;
  const int tz = tid % kTZ, ty = tid / kTZ;
  const int oy = ty + 2, oz = tz + 2;  // own cell in plane coordinates
  // the halo-2 cell this thread converts and the halo-1 cell it smooths
  const bool has_r2 = tid >= kNRing2First;
  const bool has_r1 = tid < kNRing1;
  int r2y = 0, r2z = 0, r1y = 0, r1z = 0;
  if (has_r2) nm_ring2(tid - kNRing2First, r2y, r2z);
  if (has_r1) nm_ring1(tid, r1y, r1z);
  const bool r2_in1 = has_r2 && r2y >= 1 && r2y <= kTY + 2 && r2z >= 1 &&
                      r2z <= kTZ + 2;

  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;

  for (int tile = blockIdx.x; tile < tg.ntiles; tile += gridDim.x) {
    const int tzt = tile % tg.tz_tiles;
    const int rest = tile / tg.tz_tiles;
    const int tyt = rest % tg.ty_tiles;
    const int ch = rest / tg.ty_tiles;
    const int32_t y0 = tyt * kTY - 2, z0 = tzt * kTZ - 2;  // plane origin
    const int32_t xs = tg.x0 + ch * tg.xc;
    const int32_t xe = edge ? xs + 1 : min(xs + tg.xc, tg.x1);
    const int32_t y = y0 + oy, z = z0 + oz;

    // raw inputs of plane-cell (sy, sz) of plane x into sm.raw
    auto issue_cell = [&](int32_t x, int sy, int sz) {
      bool okx, oky, okz;
      const int32_t gx = wrap(x, tg.X, tg.px, okx);
      const int32_t gy = wrap(y0 + sy, tg.Y, tg.py, oky);
      const int32_t gz = wrap(z0 + sz, tg.Z, tg.pz, okz);
      const bool ok = okx && oky && okz;
      const int64_t j = (int64_t)gx * sX + (int64_t)gy * sY + gz;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (q >= nc || !act[q]) continue;
        const int64_t o = q * n + j;
        if (!ok) {
          sm.raw[q][sy][sz] = 0.0;
          continue;
        }
        if (kClose) {
          cp_async8(&sm.raw[q][sy][sz], zin + o);
          continue;
        }
        cp_async8(&sm.raw[q][sy][sz], r + o);
        if (!(MODE == 0 && kFirst)) {
          cp_async8(&sm.raw[3 + q][sy][sz], vin + o);
          if (MODE == 0) cp_async8(&sm.raw[6 + q][sy][sz], pin + o);
        }
      }
      if (ok)
        cp_async8(&sm.raw[9][sy][sz], dinv + j);
      else
        sm.raw[9][sy][sz] = 0.0;
    };
    auto issue_plane = [&](int32_t x) {
      issue_cell(x, oy, oz);
      if (has_r2) issue_cell(x, r2y, r2z);
      cp_async_commit();
    };
    // y (undivided) and g1 = y / A of plane-cell (sy, sz)
    auto yval = [&](int sy, int sz, int q) {
      const double rr = sm.raw[q][sy][sz];
      if (kClose || (MODE == 0 && kFirst)) return rr;
      const double vv = sm.raw[3 + q][sy][sz];
      return MODE == 0 ? rr + c0[q] * (sm.raw[6 + q][sy][sz] - c1[q] * vv)
                       : rr - c0[q] * vv;
    };
    auto convert_cell = [&](int slot3, int slot2, int sy, int sz, bool in1,
                            double (&yv)[3]) {
      const double dj = sm.raw[9][sy][sz];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        yv[q] = 0.0;
        if (q >= nc || !act[q]) continue;
        yv[q] = yval(sy, sz, q);
        sm.g1[slot3][q][sy][sz] = yv[q] * dj;
      }
      if (in1) sm.dv[slot2][sy][sz] = dj;
    };
    // D^-1 N g1 at plane-cell (sy, sz) of plane x (slot3 = x % 3)
    auto smooth_cell = [&](int32_t x, int sy, int sz, const double (&cf)[6],
                           double (&out)[3]) {
      const int sm3 = mod3(x - 1), s0 = mod3(x), sp3 = mod3(x + 1);
      const double dj = sm.dv[x & 1][sy][sz];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        out[q] = 0.0;
        if (q >= nc || !act[q]) continue;
        const double h = cf[0] * sm.g1[sm3][q][sy][sz] +
                         cf[1] * sm.g1[sp3][q][sy][sz] +
                         cf[2] * sm.g1[s0][q][sy - 1][sz] +
                         cf[3] * sm.g1[s0][q][sy + 1][sz] +
                         cf[4] * sm.g1[s0][q][sy][sz - 1] +
                         cf[5] * sm.g1[s0][q][sy][sz + 1];
        out[q] = dj * h;
      }
    };
    auto in_domain = [&](int32_t x, int sy, int sz) {
      bool a1, a2, a3;
      wrap(x, tg.X, tg.px, a1);
      wrap(y0 + sy, tg.Y, tg.py, a2);
      wrap(z0 + sz, tg.Z, tg.pz, a3);
      return a1 && a2 && a3;
    };
    auto coord = [&](int32_t x, int sy, int sz, int32_t &gx, int32_t &gy,
                     int32_t &gz) {
      bool ok;
      gx = wrap(x, tg.X, tg.px, ok);
      gy = wrap(y0 + sy, tg.Y, tg.py, ok);
      gz = wrap(z0 + sz, tg.Z, tg.pz, ok);
    };

    // own-cell registers: y of planes q-2, q-1, q; q1 of planes q-3, q-1
    double ya[3] = {0, 0, 0}, yb[3] = {0, 0, 0}, yc[3] = {0, 0, 0};
    double qa[3] = {0, 0, 0}, qb[3] = {0, 0, 0}, qc[3] = {0, 0, 0};
    double cA[6] = {0, 0, 0, 0, 0, 0};  // own N row of plane q-2
    // stage-1-only passes (close, edge) smooth planes [xs, xe); the full
    // passes [xs - 1, xe], except a slab's ghost planes, whose q1 comes
    // from qghost (so the planes beyond them are never converted)
    const bool one = kClose || edge;
    const bool lo_g = qghost && xs == tg.x0, hi_g = qghost && xe == tg.x1;
    const int32_t qbeg = one || lo_g ? xs - 1 : xs - 2;
    const int32_t qconv = one || hi_g ? xe : xe + 1;  // last converted plane
    const int32_t qend = one ? xe : xe + 1;
    __syncthreads();  // the previous tile is done with every buffer
    issue_plane(qbeg);
    for (int32_t q = qbeg; q <= qend; ++q) {
      // plane q-1's N rows (own cell, halo-1 cell) and q-2's r^: plain
      // loads, consumed after the barriers
      const int32_t x1 = q - 1, x2 = q - 2;
      const bool do1 = x1 >= (one ? xs : xs - 1) && x1 <= (one ? xe - 1 : xe);
      const bool ghost1 = do1 && ((lo_g && x1 == xs - 1) || (hi_g && x1 == xe));
      const bool do2 = !one && x2 >= xs;
      double cB[6] = {0, 0, 0, 0, 0, 0}, cR[6] = {0, 0, 0, 0, 0, 0};
      bool own1 = false, ring1_ok = false;
      if (ghost1) {
        // the neighbour rank's stage 1 of this plane (own column only)
        const int64_t ig = (int64_t)x1 * sX + (int64_t)y * sY + z;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          qc[c] = (c < nc && act[c]) ? __ldg(qghost + c * n + ig) : 0.0;
      } else if (do1) {
        own1 = in_domain(x1, oy, oz);
        int32_t gx, gy, gz;
        coord(x1, oy, oz, gx, gy, gz);
        if (own1) nm_coefs<kTrans>(tg, a, n, gx, gy, gz, cB);
        if (has_r1) {
          ring1_ok = in_domain(x1, r1y, r1z);
          if (ring1_ok) {
            coord(x1, r1y, r1z, gx, gy, gz);
            nm_coefs<kTrans>(tg, a, n, gx, gy, gz, cR);
          }
        }
      }
      double rh[3] = {0, 0, 0};
      if (MODE == 0 && do2) {
        const int64_t i2 = (int64_t)x2 * sX + (int64_t)y * sY + z;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < nc && act[c]) rh[c] = __ldg(w.rhat + c * n + i2);
      }
      cp_async_wait_all();
      __syncthreads();  // B_a: plane q's raw inputs have landed everywhere
      // convert plane q
      if (q <= qconv) {
        convert_cell(mod3(q), q & 1, oy, oz, true, yc);
        if (has_r2) {
          double tmp[3];
          convert_cell(mod3(q), q & 1, r2y, r2z, r2_in1, tmp);
        }
      }
      __syncthreads();  // B_b: g1(q) complete; the raw buffer is free
      if (q + 1 <= qconv) issue_plane(q + 1);
      // stage 1 at plane q - 1
      if (do1 && !ghost1) {
        if (kClose) {
          // x += g1 - D^-1 N g1 at the own cell (tile cells only)
          smooth_cell(x1, oy, oz, cB, qc);
          const int64_t i1 = (int64_t)x1 * sX + (int64_t)y * sY + z;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (c >= nc || !act[c]) continue;
            const int64_t o = c * n + i1;
            xout[o] += sm.g1[mod3(x1)][c][oy][oz] - qc[c];
          }
        } else if (edge) {
          smooth_cell(x1, oy, oz, cB, qc);
          const int64_t i1 = (int64_t)x1 * sX + (int64_t)y * sY + z;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < nc && act[c]) qedge[c * n + i1] = qc[c];
        } else {
          smooth_cell(x1, oy, oz, cB, qc);
          if (!own1)
            for (int c = 0; c < 3; ++c) qc[c] = 0.0;
#pragma unroll
          for (int c = 0; c < 3; ++c) sm.q1[x1 & 1][c][oy][oz] = qc[c];
          if (has_r1) {
            double qr[3];
            smooth_cell(x1, r1y, r1z, cR, qr);
#pragma unroll
            for (int c = 0; c < 3; ++c)
              sm.q1[x1 & 1][c][r1y][r1z] = ring1_ok ? qr[c] : 0.0;
          }
        }
      }
      // stage 2 at plane q - 2: out = y - N q1.  Its in-plane q1 (slot
      // x2 & 1) was written in the previous step, before this step's
      // barriers; this step's stage 1 writes the other slot.
      if (do2) {
        const int64_t i2 = (int64_t)x2 * sX + (int64_t)y * sY + z;
        const int s2 = x2 & 1;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (c >= nc || !act[c]) continue;
          const double off = cA[0] * qa[c] + cA[1] * qc[c] +
                             cA[2] * sm.q1[s2][c][oy - 1][oz] +
                             cA[3] * sm.q1[s2][c][oy + 1][oz] +
                             cA[4] * sm.q1[s2][c][oy][oz - 1] +
                             cA[5] * sm.q1[s2][c][oy][oz + 1];
          const double out = ya[c] - off;
          const int64_t o = c * n + i2;
          vout[o] = out;
          if (MODE == 0) {
            pout[o] = ya[c];
            acc[c] += rh[c] * out;
          } else {
            acc[3 * c] += ya[c] * ya[c];
            acc[3 * c + 1] += out * out;
            acc[3 * c + 2] += out * ya[c];
          }
        }
      }
      // rotate the own-cell rings
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ya[c] = yb[c];
        yb[c] = yc[c];
        qa[c] = qb[c];
        qb[c] = qc[c];
      }
#pragma unroll
      for (int f = 0; f < 6; ++f) cA[f] = cB[f];
    }
    cp_async_wait_all();
  }
  if (kClose || edge) return;
  double tot[K];
  if (!grid_reduce<K>(acc, partials, counter, tot)) return;
  if (MODE == 0) {
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
  } else {
    // all_done is left alone: k_bi_xr applies the early-exit update
    for (int q = 0; q < nc; ++q) {
      CompState &c = st->c[q];
      if (!act[q]) continue;
      c.res = sqrt(tot[3 * q]);
      if (c.res <= c.tol_abs) {
        c.converged = 1;
        c.done = 1;
        c.pending = 1;
      } else if (tot[3 * q + 1] < DBL_MIN) {
        c.fail = 1;
        c.done = 1;
      } else {
        c.omega = tot[3 * q + 2] / tot[3 * q + 1];
      }
    }
  }
}
