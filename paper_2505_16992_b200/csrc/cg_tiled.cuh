// cg_tiled.cuh -- the pressure CG's direction update fused into its SpMV on
// 2.5D tiles (3D single-device boxes with whole 8 x 32 Y/Z tiles).
// Included by solvers.cu inside namespace pf (uses TileGeo, wrap, cp_async8,
// MgLevel).
//
// The reference's CG iteration (S/linalg.py:136-170) updates the direction
// p = z + beta p (after zero-mean projection) and then applies the
// operator.  Here one pass forms p' = beta p + (z - zbar) at every stencil
// point from z and the previous direction, stores p' at its own cells and
// applies the level-0 face form of K (q = sum_f w_f (p'_i - p'_nb), the
// operator k_cg_spmv_faces applies): 56 B/cell (z, p, 3 face weights in;
// p', q out) instead of the 24 + 40 of the separate direction update and
// gather SpMV, and tiled, so every array is read once per cell.  The
// directions ping-pong by iteration parity: iteration it (c.iter before this
// pass) reads P[(it & 1) ^ 1] and writes P[it & 1]; the first iteration
// forms p' = z - zbar (the reference's initial direction) and reads no p.

constexpr int kCgArr = 4;     // z, p, wy, wz
constexpr int kCgStages = 3;  // raw planes in flight (a light pass)
struct CgTileSmem {
  double raw[kCgStages][kCgArr][kTY + 2][kTZ + 2];
  double g[2][kTY + 2][kTZ + 2];  // p' of planes x & 1
};
constexpr size_t kCgTileSmem = sizeof(CgTileSmem);
constexpr int kCgMinB = 4;    // CTAs per SM (36 KB of shared memory each)

// MODE 0: the fused direction update + SpMV above.  The same tiled face
// stencil also forms the CG setup residual (MODE 1: r = bp - K x, sum r ->
// the zero-mean projection; k_cg_resid_faces) and the true-residual
// verification (MODE 2: |bp - K x|, S/linalg.py:236-239;
// k_cg_true_res_faces): z is then x, P0 / q are bp / r.
template <int MODE>
__global__ void __launch_bounds__(kTileThreads, kCgMinB)
    k_cg_tiled(TileGeo tg, MgLevel L, const double *__restrict__ z,
               double *P0, double *P1, double *__restrict__ q,
               SolverState *st, double *partials, unsigned *counter, Rng rg) {
  if (MODE != 2 && st->all_done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CgTileSmem &sm = *reinterpret_cast<CgTileSmem *>(smem_raw);
  const CompState &cs = st->c[0];
  const int it = cs.iter;
  const bool first = MODE != 0 || it == 0;
  const double beta = first ? 0.0 : cs.beta;
  const double zbar = MODE == 0 ? cs.zbar : 0.0;
  const double *__restrict__ bp = P0;
  const double *__restrict__ pold = (it & 1) ? P0 : P1;
  double *__restrict__ pnew = (it & 1) ? P1 : P0;
  const double *__restrict__ wx = L.wx;
  const double *__restrict__ wy = L.wy;
  const double *__restrict__ wz = L.wz;
  const int64_t sX = (int64_t)tg.Y * tg.Z, sY = tg.Z;
  const int tz = threadIdx.x % kTZ, ty = threadIdx.x / kTZ;

  auto issue = [&](int b, int32_t x, int32_t y, int32_t zc, int sy, int sz) {
    bool okx, oky, okz;
    x = wrap(x, tg.X, tg.px, okx);
    y = wrap(y, tg.Y, tg.py, oky);
    zc = wrap(zc, tg.Z, tg.pz, okz);
    const int64_t j = (int64_t)x * sX + (int64_t)y * sY + zc;
    if (okx && oky && okz) {
      cp_async8(&sm.raw[b][0][sy][sz], z + j);
      if (!first) cp_async8(&sm.raw[b][1][sy][sz], pold + j);
      cp_async8(&sm.raw[b][2][sy][sz], wy + j);
      cp_async8(&sm.raw[b][3][sy][sz], wz + j);
    } else {
      // outside a walled box: its face weights are zero (any finite p)
      sm.raw[b][0][sy][sz] = 0.0;
      sm.raw[b][1][sy][sz] = 0.0;
      sm.raw[b][2][sy][sz] = 0.0;
      sm.raw[b][3][sy][sz] = 0.0;
    }
  };
  auto pval = [&](int b, int sy, int sz) {
    const double zz = sm.raw[b][0][sy][sz] - zbar;
    return first ? zz : beta * sm.raw[b][1][sy][sz] + zz;
  };

  double acc[1] = {0.0};
  for (int tile = blockIdx.x; tile < tg.ntiles; tile += gridDim.x) {
    const int tzt = tile % tg.tz_tiles;
    const int rest = tile / tg.tz_tiles;
    const int tyt = rest % tg.ty_tiles;
    const int ch = rest / tg.ty_tiles;
    const int32_t y = tyt * kTY + ty, zc = tzt * kTZ + tz;
    const int32_t xs = tg.x0 + ch * tg.xc;
    const int32_t xe = min(xs + tg.xc, tg.x1);
    bool halo_cell = true;
    int hy = 0, hz = 0, sy_ = 0, sz_ = 0;
    if (threadIdx.x < 2 * kTZ) {
      const int side = threadIdx.x / kTZ;
      hy = tyt * kTY + (side ? kTY : -1);
      hz = zc;
      sy_ = side ? kTY + 1 : 0;
      sz_ = tz + 1;
    } else if (threadIdx.x < 2 * kTZ + 2 * kTY) {
      const int k = threadIdx.x - 2 * kTZ;
      const int side = k / kTY;
      hy = tyt * kTY + (k % kTY);
      hz = tzt * kTZ + (side ? kTZ : -1);
      sy_ = (k % kTY) + 1;
      sz_ = side ? kTZ + 1 : 0;
    } else {
      halo_cell = false;
    }
    auto rslot = [](int32_t x) { return (x + kCgStages) % kCgStages; };
    auto issue_plane = [&](int32_t x) {
      const int b = rslot(x);
      issue(b, x, y, zc, ty + 1, tz + 1);
      if (halo_cell) issue(b, x, hy, hz, sy_, sz_);
      cp_async_commit();
    };
    // p' of plane x (tile + halo) into g buffer x & 1; own value returned
    auto convert = [&](int32_t x) {
      const int b = rslot(x), gb2 = x & 1;
      const double pc = pval(b, ty + 1, tz + 1);
      sm.g[gb2][ty + 1][tz + 1] = pc;
      if (halo_cell) sm.g[gb2][sy_][sz_] = pval(b, sy_, sz_);
      return pc;
    };
    // X face weight of plane x at the own column (0 outside a walled box)
    auto wx_at = [&](int32_t x) {
      bool ok;
      const int32_t gx = wrap(x, tg.X, tg.px, ok);
      return ok ? __ldg(wx + (int64_t)gx * sX + (int64_t)y * sY + zc) : 0.0;
    };

    __syncthreads();  // the previous tile is done with every buffer
    double wxm = wx_at(xs - 1);
    for (int k = 0; k < kCgStages; ++k) {
      if (xs - 1 + k <= xe) issue_plane(xs - 1 + k);
      else cp_async_commit();
    }
    cp_async_wait<kCgStages - 2>();
    __syncthreads();
    double pm = pval(rslot(xs - 1), ty + 1, tz + 1);
    double pc = convert(xs);
    __syncthreads();  // raw slot of plane xs - 1 is free again
    if (xs + kCgStages - 1 <= xe) issue_plane(xs + kCgStages - 1);
    else cp_async_commit();
    for (int32_t x = xs; x < xe; ++x) {
      const int64_t i = (int64_t)x * sX + (int64_t)y * sY + zc;
      const double wxc = __ldg(wx + i);
      const int gb = x & 1, rb = rslot(x);
      // this plane's Y / Z weights of the own cell and its -y / -z
      // neighbours: plane x landed before the previous barrier, and its raw
      // slot is refilled only after the next one
      const double wyp = sm.raw[rb][2][ty + 1][tz + 1];
      const double wym = sm.raw[rb][2][ty][tz + 1];
      const double wzp = sm.raw[rb][3][ty + 1][tz + 1];
      const double wzm = sm.raw[rb][3][ty + 1][tz];
      cp_async_wait<kCgStages - 2>();  // my copies of plane x + 1 landed
      __syncthreads();  // everyone's have; p' of plane x is complete
      const double pn = convert(x + 1);
      if (x + kCgStages <= xe) issue_plane(x + kCgStages);
      else cp_async_commit();
      const double qi = wxc * (pc - pn) + wxm * (pc - pm) +
                        wyp * (pc - sm.g[gb][ty + 2][tz + 1]) +
                        wym * (pc - sm.g[gb][ty][tz + 1]) +
                        wzp * (pc - sm.g[gb][ty + 1][tz + 2]) +
                        wzm * (pc - sm.g[gb][ty + 1][tz]);
      if (MODE == 0) {
        pnew[i] = pc;
        q[i] = qi;
        acc[0] += pc * qi;
      } else {
        const double ri = bp[i] - qi;
        if (MODE == 1) {
          q[i] = ri;
          acc[0] += ri;
        } else {
          acc[0] += ri * ri;
        }
      }
      pm = pc;
      pc = pn;
      wxm = wxc;
    }
    cp_async_wait_all();
  }
  double tot[1];
  if (!grid_reduce<1>(acc, partials, counter, tot)) return;
  if (MODE == 1) {
    st->c[0].rmean = st->zero_mean ? tot[0] / rg.ng : 0.0;
    return;
  }
  if (MODE == 2) {
    st->c[0].true_res = sqrt(tot[0]);
    return;
  }
  {
    CompState &c = st->c[0];
    c.iter += 1;
    const double pap = tot[0];
    if (!finite(pap) || fabs(pap) < DBL_MIN) {
      c.fail = 1;
      c.done = 1;
      st->all_done = 1;
      return;
    }
    c.alpha = c.rz / pap;
  }
}
