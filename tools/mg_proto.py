"""NumPy prototype of the pressure multigrid preconditioner, for exploring
convergence (iteration counts) of coarsening / smoothing variants on the
channel pressure operator before touching the CUDA code.  Developer tool,
not part of the product or the tests.

    python tools/mg_proto.py --shape 64 48 64 --ratio 1.095
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def channel_operator(shape, ratio, re_tau=180.0, cfl=0.5):
    """Face weights (wx, wy, wz) of K = -P for the channel's first step."""
    from oracle import pisoref as O
    from paper_2505_16992_b200 import mesh
    from paper_2505_16992_b200.channel import reichardt_velocity
    dom = mesh.make_channel(shape, ratio=ratio)
    u, nu, _ = reichardt_velocity(dom, re_tau, device="cpu")
    u = u.numpy()
    dt = cfl * (2 * np.pi / shape[0]) / np.abs(u).max()
    c = O.assemble_momentum(dom, u, nu, dt)
    p = O.assemble_pressure(dom, 1.0 / c[0])
    w = [p[2 + 2 * a].reshape(shape).copy() for a in range(3)]
    return w


class Level:
    def __init__(self, wx, wy, wz):
        self.wx, self.wy, self.wz = wx, wy, wz
        self.shape = wx.shape
        self.n = wx.size
        sx, sy, sz = self.shape
        # Thomas factors of the Y-line matrices
        d = self.diag()
        lo = np.concatenate([np.zeros((sx, 1, sz)), wy[:, :-1]], axis=1)
        self.ivd = np.empty_like(d)
        self.cp = np.empty_like(d)
        self.pinned = sx == 1 and sz == 1
        cprev = np.zeros((sx, sz))
        for y in range(sy):
            if self.pinned and y == sy - 1:
                self.ivd[:, y] = 1.0
                self.cp[:, y] = 0.0
                break
            iv = 1.0 / (d[:, y] + lo[:, y] * cprev)
            self.ivd[:, y] = iv
            self.cp[:, y] = -wy[:, y] * iv
            cprev = self.cp[:, y]

    def diag(self):
        wx, wy, wz = self.wx, self.wy, self.wz
        return (wx + np.roll(wx, 1, 0) + wz + np.roll(wz, 1, 2) + wy
                + np.concatenate([np.zeros_like(wy[:, :1]), wy[:, :-1]], 1))

    def apply(self, v):
        wx, wy, wz = self.wx, self.wy, self.wz
        out = np.zeros_like(v)
        f = wx * (v - np.roll(v, -1, 0))
        out += f - np.roll(f, 1, 0)
        f = wz * (v - np.roll(v, -1, 2))
        out += f - np.roll(f, 1, 2)
        f = wy[:, :-1] * (v[:, :-1] - v[:, 1:])
        out[:, :-1] += f
        out[:, 1:] -= f
        return out

    def line_solve(self, r):
        sx, sy, sz = self.shape
        lo = np.concatenate([np.zeros((sx, 1, sz)), self.wy[:, :-1]], axis=1)
        t = np.empty_like(r)
        dp = np.zeros((sx, sz))
        for y in range(sy):
            if self.pinned and y == sy - 1:
                t[:, y] = 0.0
                dp = t[:, y]
                continue
            dp = (r[:, y] + lo[:, y] * dp) * self.ivd[:, y]
            t[:, y] = dp
        z = np.empty_like(r)
        zn = np.zeros((sx, sz))
        for y in range(sy - 1, -1, -1):
            zn = t[:, y] - self.cp[:, y] * zn
            z[:, y] = zn
        return z


def aggregate(F, f):
    fx, fy, fz = f
    sx, sy, sz = F.shape
    C = (sx // fx, sy // fy, sz // fz)

    def fold(w, keep_axis):
        # fine faces crossing coarse faces of keep_axis: the last fine
        # layer of each aggregate along that axis, summed over the others
        sl = [slice(None)] * 3
        fa = f[keep_axis]
        sl[keep_axis] = slice(fa - 1, None, fa)
        v = w[tuple(sl)]
        shp = list(v.shape)
        rs = []
        for a in range(3):
            if a == keep_axis:
                rs += [shp[a], 1]
            else:
                rs += [shp[a] // f[a], f[a]]
        return v.reshape(rs).sum(axis=(1, 3, 5))

    wx = fold(F.wx, 0) if C[0] > 1 else np.zeros(C)
    wy = fold(F.wy, 1)
    wz = fold(F.wz, 2) if C[2] > 1 else np.zeros(C)
    return Level(wx, wy, wz)


def restrict(F, C, r):
    f = [F.shape[a] // C.shape[a] for a in range(3)]
    sx, sy, sz = C.shape
    return r.reshape(sx, f[0], sy, f[1], sz, f[2]).sum(axis=(1, 3, 5))


def prolong(F, C, x):
    f = [F.shape[a] // C.shape[a] for a in range(3)]
    for a in range(3):
        x = np.repeat(x, f[a], axis=a)
    return x


def build_hierarchy(w, policy, max_levels=16):
    levels = [Level(*w)]
    while len(levels) < max_levels:
        L = levels[-1]
        f = policy(L, len(levels) - 1)
        if f is None:
            break
        levels.append(aggregate(L, f))
    return levels


def policy_full(L, k):
    sx, sy, sz = L.shape
    fx = 2 if sx % 2 == 0 else 1
    fz = 2 if sz % 2 == 0 else 1
    fy = 2 if sy % 2 == 0 and sy > 2 else 1
    if fx == 1 and fz == 1:
        return None
    return fx, fy, fz


def policy_strength(thresh=0.5, y_mode="full"):
    """Coarsen X / Z only where coupling is strong relative to the
    strongest of the two (semi-coarsening of the strong direction)."""
    def pol(L, k):
        sx, sy, sz = L.shape
        sxw = L.wx.mean() if sx > 1 else 0.0
        szw = L.wz.mean() if sz > 1 else 0.0
        m = max(sxw, szw)
        fx = 2 if sx % 2 == 0 and sxw >= thresh * m else 1
        fz = 2 if sz % 2 == 0 and szw >= thresh * m else 1
        if fx == 1 and fz == 1:
            fx = 2 if sx % 2 == 0 else 1
            fz = 2 if sz % 2 == 0 else 1
        if fx == 1 and fz == 1:
            return None
        if y_mode == "full":
            fy = 2 if sy % 2 == 0 and sy > 2 else 1
        elif y_mode == "with_x":
            fy = 2 if sy % 2 == 0 and sy > 2 and fx == 2 else 1
        else:
            fy = 1
        return fx, fy, fz
    return pol


def coarse_solve(L, r):
    if L.pinned:
        z = L.line_solve(r)
        return z - z.mean()
    return None


def kcycle(levels, k, r, **kw):
    """Two flexible-CG steps preconditioned by the cycle at level k
    (Notay's K-cycle)."""
    L = levels[k]
    c1 = vcycle(levels, k, r, **kw)
    v1 = L.apply(c1)
    rho1 = (c1 * v1).sum()
    a1 = (c1 * r).sum()
    r2 = r - (a1 / rho1) * v1
    if np.linalg.norm(r2) <= 0.25 * np.linalg.norm(r):
        return (a1 / rho1) * c1
    c2 = vcycle(levels, k, r2, **kw)
    v2 = L.apply(c2)
    g = (c2 * v1).sum()
    beta = (c2 * v2).sum() - g * g / rho1
    a2 = (c2 * r2).sum()
    return (a1 / rho1 - g * a2 / (rho1 * beta)) * c1 + (a2 / beta) * c2


def vcycle(levels, k, r, omega, nu1=1, nu2=1, alpha=1.0, gamma=1,
           coarse_sweeps=5, kc_levels=()):
    kw = dict(omega=omega, nu1=nu1, nu2=nu2, alpha=alpha, gamma=gamma,
              coarse_sweeps=coarse_sweeps, kc_levels=kc_levels)
    L = levels[k]
    if k == len(levels) - 1:
        z = coarse_solve(L, r)
        if z is not None:
            return z
        z = omega * L.line_solve(r)
        for _ in range(coarse_sweeps - 1):
            z += omega * L.line_solve(r - L.apply(z))
        return z
    C = levels[k + 1]
    z = omega * L.line_solve(r)
    for _ in range(nu1 - 1):
        z += omega * L.line_solve(r - L.apply(z))
    rc = restrict(L, C, r - L.apply(z))
    if k + 1 in kc_levels and k + 1 < len(levels) - 1:
        zc = kcycle(levels, k + 1, rc, **kw)
    else:
        zc = np.zeros(C.shape)
        for _ in range(gamma):
            zc += vcycle(levels, k + 1, rc - (C.apply(zc) if _ else 0), **kw)
    z += alpha * prolong(L, C, zc)
    for _ in range(nu2):
        z += omega * L.line_solve(r - L.apply(z))
    return z


def pcg(levels, b, tol=1e-8, maxiter=500, **kw):
    L = levels[0]
    b = b - b.mean()
    x = np.zeros_like(b)
    r = b.copy()
    bn = np.linalg.norm(b)
    z = vcycle(levels, 0, r, **kw)
    z -= z.mean()
    p = z.copy()
    rz = (r * z).sum()
    for it in range(1, maxiter + 1):
        q = L.apply(p)
        a = rz / (p * q).sum()
        x += a * p
        r_old = r.copy()
        r -= a * q
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = vcycle(levels, 0, r, **kw)
        z -= z.mean()
        rz2 = (r * z).sum()
        # flexible (Polak-Ribiere) beta: robust to a varying preconditioner
        p = z + ((z * (r - r_old)).sum() / rz) * p
        rz = rz2
    return maxiter


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[64, 48, 64])
    ap.add_argument("--ratio", type=float, default=1.095)
    ap.add_argument("--cfl", type=float, default=0.5)
    args = ap.parse_args()
    t0 = time.time()
    w = channel_operator(tuple(args.shape), args.ratio, cfl=args.cfl)
    print(f"operator {time.time() - t0:.1f}s; mean wx wy wz",
          [float(v.mean()) for v in w])
    rng = np.random.default_rng(0)
    b = rng.standard_normal(tuple(args.shape))
    variants = {
        "full w.85": (policy_full, dict(omega=0.85)),
        "full w.7": (policy_full, dict(omega=0.7)),
        "full w1.0": (policy_full, dict(omega=1.0)),
        "full K@1": (policy_full, dict(omega=0.85, kc_levels=(1,))),
        "full K@1,2": (policy_full, dict(omega=0.85, kc_levels=(1, 2))),
        "full K@all": (policy_full, dict(omega=0.85,
                                         kc_levels=tuple(range(1, 16)))),
        "full K@2+": (policy_full, dict(omega=0.85,
                                        kc_levels=tuple(range(2, 16)))),
        "strength.5 K@all": (policy_strength(0.5),
                             dict(omega=0.85, kc_levels=tuple(range(1, 16)))),
    }
    only = os.environ.get("VARIANTS")
    for name, (pol, kw) in variants.items():
        if only and name not in only.split(";"):
            continue
        lv = build_hierarchy(w, pol)
        t0 = time.time()
        it = pcg(lv, b, **kw)
        print(f"{name:22s} levels {[l.shape for l in lv]} iters {it} "
              f"({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()


class FFTPrecond:
    """Exact inverse of the XZ-plane-averaged operator: Fourier in the
    periodic X and Z, tridiagonal in Y per wavenumber pair."""

    def __init__(self, w):
        wx, wy, wz = w
        sx, sy, sz = wx.shape
        self.shape = wx.shape
        ax = wx.mean(axis=(0, 2))            # (sy,)
        az = wz.mean(axis=(0, 2))
        ay = wy.mean(axis=(0, 2))            # face y | y+1 (last = 0)
        kx = np.arange(sx)[:, None]
        kz = np.arange(sz // 2 + 1)[None, :]
        lx = 2.0 - 2.0 * np.cos(2 * np.pi * kx / sx)
        lz = 2.0 - 2.0 * np.cos(2 * np.pi * kz / sz)
        self.lo = np.concatenate([[0.0], ay[:-1]])
        self.up = ay
        self.d = (ax[None, :, None] * lx[:, None, :] + az[None, :, None]
                  * lz[:, None, :] + (self.lo + self.up)[None, :, None])
        self.sy = sy

    def __call__(self, r):
        rh = np.fft.rfft2(r, axes=(0, 2))    # (sx, sy, sz//2+1)
        d = self.d.astype(complex).copy()
        sy = self.sy
        # pin the singular (0,0) mode's last row
        zero = np.zeros(d.shape[0:1] + d.shape[2:], bool)
        zero[0, 0] = True
        # Thomas along y
        cp = np.zeros(d.shape, complex)
        dp = np.zeros(d.shape, complex)
        for y in range(sy):
            den = d[:, y] + (self.lo[y] * cp[:, y - 1] if y else 0.0)
            rr = rh[:, y] + (self.lo[y] * dp[:, y - 1] if y else 0.0)
            if y == sy - 1:
                den = np.where(zero, 1.0, den)
                rr = np.where(zero, 0.0, rr)
            cp[:, y] = -self.up[y] / den
            dp[:, y] = rr / den
        z = np.zeros_like(rh)
        zn = 0.0
        for y in range(sy - 1, -1, -1):
            zn = dp[:, y] - cp[:, y] * zn
            z[:, y] = zn
        out = np.fft.irfft2(z, s=(self.shape[0], self.shape[2]), axes=(0, 2))
        return out - out.mean()


def pcg_fn(L, M, b, tol=1e-8, maxiter=500):
    b = b - b.mean()
    x = np.zeros_like(b)
    r = b.copy()
    bn = np.linalg.norm(b)
    z = M(r)
    p = z.copy()
    rz = (r * z).sum()
    for it in range(1, maxiter + 1):
        q = L.apply(p)
        a = rz / (p * q).sum()
        x += a * p
        r -= a * q
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = M(r)
        rz2 = (r * z).sum()
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxiter
