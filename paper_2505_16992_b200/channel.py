"""Turbulent-channel drivers (mirror of S/piso.py:512-546, 661-745).

``reichardt_init`` builds the channel initial condition exactly as the
reference does (law-of-the-wall mean profile plus a smoothed, windowed,
discretely solenoidal random perturbation), ``wall_forcing_source`` the
per-step streamwise body force that balances the mean wall shear, and
``adaptive_dt`` the CFL time step.  They are the callers on either side of
the step (SURVEY.md §8 f, rank 2).

Single-block box domains (the channel) run on the device with torch tensor
arithmetic in the reference's operation order; other domains use the host
neighbour tables.  The random field is drawn with NumPy's
``default_rng(seed)`` so a given seed reproduces the reference's field.
"""

import numpy as np
import torch

from .piso import F64, FlowState, bc_soa, bc_views, make_state


def reichardt_profile(y_plus, kappa=0.41):
    """Smooth law-of-the-wall profile in wall units (S/piso.py:661-665)."""
    if torch.is_tensor(y_plus):
        return (torch.log1p(kappa * y_plus) / kappa
                + 7.8 * (1.0 - torch.exp(-y_plus / 11.0)
                         - (y_plus / 11.0) * torch.exp(-y_plus / 3.0)))
    y_plus = np.asarray(y_plus, dtype=np.float64)
    return (np.log1p(kappa * y_plus) / kappa
            + 7.8 * (1.0 - np.exp(-y_plus / 11.0)
                     - (y_plus / 11.0) * np.exp(-y_plus / 3.0)))


def _wall_layer(domain, wall_axis):
    """Cell distance to the nearest end of the wall axis, per block
    (S/piso.py:717-729)."""
    layer = np.empty(domain.n, dtype=np.int64)
    for b in range(len(domain.blocks)):
        shape = domain.block_shapes[b]
        m = shape[wall_axis]
        idx = np.arange(m)
        lay = np.minimum(idx, m - 1 - idx)
        sh = [1] * len(shape)
        sh[wall_axis] = m
        lo, hi = domain.offsets[b], domain.offsets[b + 1]
        layer[lo:hi] = np.broadcast_to(lay.reshape(sh), shape).reshape(-1)
    return layer


class _BoxOps:
    """Neighbour fetches on a single box block with torch (device)."""

    def __init__(self, domain, device):
        self.shape, self.periodic = domain.box_layout()
        self.d = domain.dim
        self.device = device

    def fetch(self, f, a, s):
        """(nb value, has-neighbour mask) of a (*shape, k) field along axis
        a, side s."""
        sh = self.shape
        if self.periodic[a]:
            return torch.roll(f, shifts=-1 if s else 1, dims=a), None
        nb = torch.roll(f, shifts=-1 if s else 1, dims=a)
        idx = torch.arange(sh[a], device=self.device)
        ok = (idx < sh[a] - 1) if s else (idx > 0)
        view = [1] * len(f.shape)
        view[a] = sh[a]
        return nb, ok.reshape(view)

    def mirror_grad(self, phi):
        """wide_grad(phi, 'mirror') of a (*shape) field -> (*shape, d)."""
        out = []
        for a in range(self.d):
            hi, mh = self.fetch(phi, a, 1)
            lo, ml = self.fetch(phi, a, 0)
            vhi = hi if mh is None else torch.where(mh, hi, phi)
            vlo = lo if ml is None else torch.where(ml, lo, phi)
            out.append(0.5 * (vhi - vlo))
        return torch.stack(out, dim=-1)


def reichardt_init(domain, re_tau, delta=1.0, wall_axis=1, flow_axis=0,
                   perturbation=0.1, seed=0, device=None):
    """Channel initial state (S/piso.py:668-714).  Returns
    (state, nu, u_tau)."""
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if device is None else torch.device(device)
    u, nu, u_tau = reichardt_velocity(domain, re_tau, delta, wall_axis,
                                      flow_axis, perturbation, seed, dev)
    return make_state(domain, u0=u, device=dev), nu, u_tau


def reichardt_velocity(domain, re_tau, delta=1.0, wall_axis=1, flow_axis=0,
                       perturbation=0.1, seed=0, device="cpu"):
    """The (n, d) initial velocity of :func:`reichardt_init` as a tensor on
    ``device`` (any torch device), plus (nu, u_tau)."""
    dev = torch.device(device)
    n, d = domain.n, domain.dim
    re_cl = (re_tau / 0.116) ** (1.0 / 0.88)
    nu = delta / re_cl
    u_tau = re_tau * nu / delta
    box = domain.box_layout()
    sep = domain.separable_metrics()
    if box is None or sep is None:
        u = _reichardt_host(domain, re_tau, nu, u_tau, delta, wall_axis,
                            flow_axis, perturbation, seed)
        return torch.as_tensor(u, dtype=F64, device=dev), nu, u_tau
    shape = box[0]
    ops = _BoxOps(domain, dev)
    coords = domain._separable[0]
    y1 = 0.5 * (coords[wall_axis][:-1] + coords[wall_axis][1:])
    yv = torch.as_tensor(y1, dtype=F64, device=dev)
    view = [1] * d
    view[wall_axis] = shape[wall_axis]
    y = yv.reshape(view).expand(*shape)
    dist = torch.minimum(y, 2.0 * delta - y)
    y_plus = torch.clamp(dist, min=0.0) * u_tau / nu
    u = torch.zeros(shape + (d,), dtype=F64, device=dev)
    u[..., flow_axis] = u_tau * reichardt_profile(y_plus)
    if perturbation:
        rng = np.random.default_rng(seed)
        n_psi = 3 if d == 3 else 1
        psi = torch.as_tensor(rng.standard_normal((n, n_psi)), dtype=F64,
                              device=dev).reshape(shape + (n_psi,))
        for _ in range(2):
            for a in range(d):
                hi, mh = ops.fetch(psi, a, 1)
                lo, ml = ops.fetch(psi, a, 0)
                if mh is not None:
                    hi = torch.where(mh, hi, psi)
                    lo = torch.where(ml, lo, psi)
                psi = 0.5 * psi + 0.25 * (hi + lo)
        layer = torch.as_tensor(_wall_layer(domain, wall_axis),
                                device=dev).reshape(shape)
        window = torch.where(layer >= 2,
                             torch.sin(np.pi * dist / (2 * delta)) ** 2,
                             torch.zeros((), dtype=F64, device=dev))
        psi = psi * window.unsqueeze(-1)
        grads = [ops.mirror_grad(psi[..., c]) for c in range(n_psi)]
        if d == 2:
            g = grads[0]
            uflux = torch.stack([g[..., 1], -g[..., 0]], dim=-1)
        else:
            gx, gy, gz = grads
            uflux = torch.stack([gz[..., 1] - gy[..., 2],
                                 gx[..., 2] - gz[..., 0],
                                 gy[..., 0] - gx[..., 1]], dim=-1)
        dxs = []
        for a in range(d):
            vw = [1] * d
            vw[a] = shape[a]
            dxs.append(torch.as_tensor(sep[a], dtype=F64,
                                       device=dev).reshape(vw).expand(*shape))
        jac = dxs[0]
        for a in range(1, d):
            jac = jac * dxs[a]
        du = torch.stack([dxs[a] * uflux[..., a] for a in range(d)],
                         dim=-1) / jac.unsqueeze(-1)
        peak = float(du.abs().max())
        if peak > 0:
            du = du * (perturbation * u_tau
                       * float(reichardt_profile(np.array([re_tau]))[0])
                       / peak)
        u = u + du
    return u.reshape(n, d), nu, u_tau


def _reichardt_host(domain, re_tau, nu, u_tau, delta, wall_axis, flow_axis,
                    perturbation, seed):
    n, d = domain.n, domain.dim
    y = domain.centers[:, wall_axis]
    dist = np.minimum(y, 2.0 * delta - y)
    y_plus = np.maximum(dist, 0.0) * u_tau / nu
    u = np.zeros((n, d))
    u[:, flow_axis] = u_tau * reichardt_profile(y_plus)
    if not perturbation:
        return u
    rng = np.random.default_rng(seed)
    n_psi = 3 if d == 3 else 1
    psi = rng.standard_normal((n, n_psi))
    for _ in range(2):
        for a in range(d):
            hi, lo = domain.nbr[a, 1], domain.nbr[a, 0]
            psi = 0.5 * psi + 0.25 * (
                np.where((hi >= 0)[:, None], psi[np.maximum(hi, 0)], psi)
                + np.where((lo >= 0)[:, None], psi[np.maximum(lo, 0)], psi))
    layer = _wall_layer(domain, wall_axis)
    window = np.where(layer >= 2, np.sin(np.pi * dist / (2 * delta)) ** 2, 0.0)
    psi = psi * window[:, None]

    def mgrad(phi):
        g = np.empty((n, d))
        for a in range(d):
            hi, lo = domain.nbr[a, 1], domain.nbr[a, 0]
            g[:, a] = 0.5 * (np.where(hi >= 0, phi[np.maximum(hi, 0)], phi)
                             - np.where(lo >= 0, phi[np.maximum(lo, 0)], phi))
        return g

    grads = [mgrad(psi[:, c]) for c in range(n_psi)]
    if d == 2:
        uflux = np.stack([grads[0][:, 1], -grads[0][:, 0]], axis=-1)
    else:
        gx, gy, gz = grads
        uflux = np.stack([gz[:, 1] - gy[:, 2], gx[:, 2] - gz[:, 0],
                          gy[:, 0] - gx[:, 1]], axis=-1)
    du = np.einsum("nij,nj->ni", domain.dxdxi, uflux) / domain.jac[:, None]
    peak = np.abs(du).max()
    if peak > 0:
        du *= perturbation * u_tau * reichardt_profile(
            np.array([re_tau])).item() / peak
    return u + du


class WallForcing:
    """Per-step streamwise forcing nu <|u/dist|>_walls / delta
    (wall_shear_mean / wall_forcing_source, S/piso.py:523-542), evaluated on
    the device from the first cell row next to every Dirichlet wall."""

    def __init__(self, domain, device, wall_axis=1, flow_axis=0, delta=1.0,
                 owned=None, counts=None):
        """owned: optional (lo, hi) cell range the rows are restricted to,
        counts: the per-wall row sizes to divide by (slab.SlabWallForcing:
        the rank's owned cells, the global sizes)."""
        self.flow_axis = flow_axis
        self.delta = delta
        self.d = domain.dim
        walls = [f for f in domain.bfaces
                 if f.kind == "dirichlet" and f.axis == wall_axis]
        if not walls:
            raise ValueError("no wall faces on that axis")
        cells, dists, seg = [], [], [0]
        for f in walls:
            cen = domain._cell_centres_of(
                next(b for b in range(len(domain.blocks))
                     if domain.offsets[b] <= f.cells[0]
                     < domain.offsets[b + 1]), f.cells)
            dist = np.linalg.norm(cen - f.face_centers, axis=1)
            c = np.asarray(f.cells)
            if owned is not None:
                keep = (c >= owned[0]) & (c < owned[1])
                c, dist = c[keep], dist[keep]
            dists.append(dist)
            cells.append(c)
            seg.append(seg[-1] + len(c))
        self.domain = domain
        self.cells = torch.as_tensor(np.concatenate(cells).astype(np.int32),
                                     device=device)
        self.dist = torch.as_tensor(np.concatenate(dists), dtype=F64,
                                    device=device)
        self.seg = torch.as_tensor(np.asarray(seg, dtype=np.int32),
                                   device=device)
        sizes = np.diff(seg).astype(np.float64) if counts is None \
            else np.asarray(counts, dtype=np.float64)
        self.cnt = torch.as_tensor(sizes, dtype=F64, device=device)
        self.nwall, self.m = len(walls), seg[-1]

    def __call__(self, u, nu):
        """(d,) device tensor source for the step whose input is u (n, d):
        one fused reduction kernel (pf_wall_forcing)."""
        from . import _lib
        from .piso import soa
        plan = self.domain.device_plan(u.device)
        out = torch.empty(self.d, dtype=F64, device=plan.device)
        _lib.call("pf_wall_forcing", plan.handle,
                  _lib.ptr(soa(u, self.domain.n, self.d, plan.device)),
                  self.flow_axis, _lib.ptr(self.cells), _lib.ptr(self.dist),
                  _lib.ptr(self.seg), _lib.ptr(self.cnt), self.nwall, self.m,
                  float(nu),
                  float(self.delta), _lib.ptr(out), _lib.ptr(plan.workspace),
                  plan.stream)
        return out


def wall_forcing_source(domain, u, nu, wall_axis=1, flow_axis=0, delta=1.0):
    """Streamwise body force balancing the mean wall shear
    (S/piso.py:535-542); returns a (d,) tensor on u's device."""
    return WallForcing(domain, u.device, wall_axis, flow_axis, delta)(u, nu)


def adaptive_dt(domain, u, cfl_max, dt_max, remaining=None):
    """Largest dt with sum_a |U^a| / J <= cfl_max (S/piso.py:512-520)."""
    from . import _lib
    from .piso import soa
    plan = domain.device_plan(u.device)
    # one fused kernel over the owned cells (pf_cfl_peak); on slab plans
    # its reduction spans the ranks, so every rank takes the same dt
    peak_t = torch.empty(1, dtype=F64, device=plan.device)
    _lib.call("pf_cfl_peak", plan.handle,
              _lib.ptr(soa(u, domain.n, domain.dim, plan.device)),
              _lib.ptr(plan.workspace), _lib.ptr(peak_t), plan.stream)
    peak = float(peak_t.item())
    dt = dt_max if peak == 0.0 else min(dt_max, cfl_max / peak)
    if remaining is not None:
        dt = min(dt, remaining)
    return dt


__all__ = ["reichardt_profile", "reichardt_init", "reichardt_velocity",
           "WallForcing",
           "wall_forcing_source", "adaptive_dt"]
