"""Channel statistics and the statistics loss on the device (SURVEY.md §8 f,
rank 1; mirror of S/stats.py:206-614).

The turbulent-channel training runs of the paper score a
rollout by its wall-normal statistics: per slice (index along the wall
axis) the mean velocity and its central covariance over the homogeneous
planes, for every frame and over the rollout window.  Here

* :func:`frame_profile` / :func:`frame_profile_backward` run in
  ``libpisob200.so`` (``pf_slice_moments``, ``pf_slice_moments_backward``):
  one fixed-order two-pass reduction per frame, no host round trip, and on
  slab domains the slices span every rank (the library adds the ranks' sums);
* :func:`window_profile`, :func:`window_profile_backward`,
  :func:`stats_loss` and :func:`stats_loss_grad` act on the small (Y, d) /
  (Y, d, d) profile tensors on the same device;
* :class:`FrameProfile` makes the profile a ``torch.autograd`` function, so
  a training loss built from it back-propagates through the discrete adjoint
  of the PISO step (``autograd.piso_step_fn``);
* :class:`ChannelAccumulator` streams per-slice means, covariances, third and
  fourth moments over frames (skewness / flatness profiles) with the exact
  pairwise merge of central moments.

Signatures, conventions (population moments, loss weights, window
semantics) and error behaviour follow the reference.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

F64 = torch.float64


# ---------------------------------------------------------------------------
# slices


@dataclass
class ChannelSlices:
    """Wall-normal slicing of a single-block channel (S/stats.py:206-231).
    ``idx`` holds the (local) cells of each slice; ``m`` is the number of
    cells per slice over the whole channel (all slab ranks)."""
    wall_axis: int
    y: np.ndarray          # (Y,) slice center coordinates
    idx: np.ndarray        # (Y, M_local) cell indices per slice (owned)
    inv: np.ndarray        # (n,) slice index of each cell (-1: ghost)
    y_lo: float            # wall coordinates
    y_hi: float
    m_total: int = 0
    domain: object = None

    @property
    def ny(self):
        return self.y.shape[0]

    @property
    def m(self):
        return self.m_total or self.idx.shape[1]

    @property
    def delta(self):
        return 0.5 * (self.y_hi - self.y_lo)

    @property
    def dy(self):
        edges = np.empty(self.ny + 1)
        edges[0], edges[-1] = self.y_lo, self.y_hi
        edges[1:-1] = 0.5 * (self.y[1:] + self.y[:-1])
        return np.diff(edges)


def channel_slices(domain, wall_axis=1):
    """Wall-normal slicing for a single-block channel (S/stats.py:234-259).
    The homogeneous axes must be periodic (no boundary faces) and both
    wall-axis sides must be prescribed walls."""
    if len(domain.block_shapes) != 1:
        raise ValueError("channel statistics need a single-block mesh")
    sides = set()
    for f in domain.bfaces:
        if f.axis != wall_axis:
            raise ValueError("homogeneous axes must be periodic")
        sides.add(f.side)
    if sides != {0, 1}:
        raise ValueError("both walls of the channel must be boundaries")
    grid = domain.block_index_grid(0)
    owned = np.ones(grid.shape, dtype=bool)
    m_total = 0
    if getattr(domain, "slab_info", None) is not None:
        owned[0] = False
        owned[-1] = False
    ny = grid.shape[wall_axis]
    idx_all = np.moveaxis(grid, wall_axis, 0).reshape(ny, -1)
    own = np.moveaxis(owned, wall_axis, 0).reshape(ny, -1)
    idx = np.stack([idx_all[j][own[j]] for j in range(ny)])
    y = domain.centers[idx, wall_axis].mean(axis=1)
    inv = np.full(domain.n, -1, dtype=np.int64)
    for j in range(ny):
        inv[idx[j]] = j
    if getattr(domain, "slab_info", None) is not None:
        m_total = idx.shape[1] * domain.nx // domain.nxl
    walls = {f.side: float(f.face_centers[:, wall_axis].mean())
             for f in domain.bfaces}
    y_lo, y_hi = sorted(walls.values())
    return ChannelSlices(wall_axis, y, idx, inv, y_lo, y_hi,
                         m_total=m_total, domain=domain)


def _plan(sl, dev):
    if sl.domain is None:
        raise ValueError("these slices carry no domain (use channel_slices)")
    return sl.domain.device_plan(dev)


def _soa(u, n, d, dev):
    from .piso import soa
    return soa(u, n, d, dev)


# ---------------------------------------------------------------------------
# per-frame profiles (device kernels)


def frame_moments(sl, u, higher=False):
    """(mean (Y, d), cov (Y, d, d)[, m3 (Y, d), m4 (Y, d)]) of a velocity
    frame (n, d) on the device."""
    dev = u.device
    _lib.require_cuda(dev)
    plan = _plan(sl, dev)
    n, d = sl.domain.n, sl.domain.dim
    us = _soa(u, n, d, dev)
    ny = sl.ny
    mean = torch.empty((ny, d), dtype=F64, device=dev)
    cov = torch.empty((ny, d, d), dtype=F64, device=dev)
    m3 = torch.empty((ny, d), dtype=F64, device=dev) if higher else None
    m4 = torch.empty((ny, d), dtype=F64, device=dev) if higher else None
    _lib.call("pf_slice_moments", plan.handle, _lib.ptr(us), sl.wall_axis,
              _lib.ptr(mean), _lib.ptr(cov), _lib.ptr(m3), _lib.ptr(m4),
              _lib.ptr(plan.workspace), plan.stream)
    return (mean, cov, m3, m4) if higher else (mean, cov)


def frame_profile(sl, u):
    """(mean, cov) slice profile of a single velocity frame
    (S/stats.py:275-278)."""
    return frame_moments(sl, u)


def slice_mean(sl, f):
    """Per-slice mean of a per-cell (n, d) velocity field over the
    homogeneous directions (S/stats.py:262-264)."""
    return frame_moments(sl, f)[0]


def slice_cov(sl, u, mean=None):
    """Per-slice central covariance (Y, d, d) (S/stats.py:267-272); the
    means are recomputed on the device (``mean`` is accepted for signature
    compatibility)."""
    return frame_moments(sl, u)[1]


def frame_profile_backward(sl, u, d_mean, d_cov):
    """Cotangent of frame_profile back onto the velocity field
    (S/stats.py:281-290): (n, d), zero on ghost planes."""
    dev = u.device
    plan = _plan(sl, dev)
    n, d = sl.domain.n, sl.domain.dim
    us = _soa(u, n, d, dev)
    mean = frame_moments(sl, u)[0]
    dm = torch.as_tensor(d_mean, dtype=F64, device=dev).contiguous()
    dc = torch.as_tensor(d_cov, dtype=F64, device=dev).contiguous()
    du = torch.zeros((d, n), dtype=F64, device=dev)
    _lib.call("pf_slice_moments_backward", plan.handle, _lib.ptr(us),
              sl.wall_axis, _lib.ptr(mean), _lib.ptr(dm), _lib.ptr(dc),
              _lib.ptr(du), plan.stream)
    return du.t()


class FrameProfile(torch.autograd.Function):
    """(mean, cov) = frame_profile(sl, u) as a differentiable function of
    the (n, d) velocity tensor."""

    @staticmethod
    def forward(ctx, u, sl):
        mean, cov = frame_profile(sl, u.detach())
        ctx.sl = sl
        ctx.save_for_backward(u.detach())
        return mean, cov

    @staticmethod
    def backward(ctx, d_mean, d_cov):
        (u,) = ctx.saved_tensors
        if d_mean is None:
            d_mean = torch.zeros((ctx.sl.ny, u.shape[1]), dtype=F64,
                                 device=u.device)
        if d_cov is None:
            d_cov = torch.zeros((ctx.sl.ny, u.shape[1], u.shape[1]),
                                dtype=F64, device=u.device)
        return frame_profile_backward(ctx.sl, u, d_mean, d_cov), None


def frame_profile_fn(sl, u):
    return FrameProfile.apply(u, sl)


# ---------------------------------------------------------------------------
# window profiles and the statistics loss (small (Y, d) tensors)


def _t(x, dev=None):
    return x if torch.is_tensor(x) else torch.as_tensor(
        np.asarray(x, dtype=np.float64), device=dev)


def window_profile(profiles):
    """Window-averaged (mean, cov) from per-frame profiles
    (S/stats.py:293-304): pooling all frames' cells per slice."""
    means = torch.stack([_t(m) for m, _ in profiles])
    covs = torch.stack([_t(c) for _, c in profiles])
    mu = means.mean(dim=0)
    dev = means - mu
    cov = covs.mean(dim=0) + torch.einsum("tyi,tyj->yij", dev, dev) / len(
        profiles)
    return mu, cov


def window_profile_backward(profiles, d_mu, d_cov):
    """Cotangents of window_profile w.r.t. each frame's (mean, cov)
    (S/stats.py:307-320)."""
    means = torch.stack([_t(m) for m, _ in profiles])
    nt = means.shape[0]
    mu = means.mean(dim=0)
    dev = means - mu
    d_mu, d_cov = _t(d_mu, means.device), _t(d_cov, means.device)
    sym = d_cov + d_cov.transpose(1, 2)
    out = []
    for t in range(nt):
        dm = d_mu / nt + torch.einsum("yij,yj->yi", sym, dev[t]) / nt
        out.append((dm, d_cov / nt))
    return out


@dataclass
class LossWeights:
    """Nonnegative weights for the statistics loss (S/stats.py:534-548)."""
    mean: np.ndarray
    cov: np.ndarray
    frame: float = 0.5
    source: float = 1.0
    div: float = 1e-4
    weight_decay: float = 0.0

    def __post_init__(self):
        self.mean = np.asarray(self.mean, dtype=np.float64)
        self.cov = np.asarray(self.cov, dtype=np.float64)
        if (self.mean < 0).any() or (self.cov < 0).any() or self.frame < 0 \
                or self.source < 0 or self.div < 0 or self.weight_decay < 0:
            raise ValueError("loss weights must be nonnegative")


def tcf_default_weights(dim=3):
    """Weight set of the turbulent-channel training runs
    (S/stats.py:551-559)."""
    mean = np.ones(dim)
    mean[1:] = 0.5
    cov = np.zeros((dim, dim))
    np.fill_diagonal(cov, 1.0)
    if dim >= 2:
        cov[0, 1] = cov[1, 0] = 1.0
    return LossWeights(mean=mean, cov=cov, frame=0.5, source=1.0, div=1e-4)


def _term(mean, cov, ref_mean, ref_cov, wm, wc):
    lm = torch.sum(wm * ((mean - ref_mean) ** 2).mean(dim=0))
    lc = torch.sum(wc * ((cov - ref_cov) ** 2).mean(dim=0))
    return lm + lc


def stats_loss_grad(profiles, reference, weights, window=None):
    """stats_loss value plus its gradients w.r.t. each frame's profile
    (S/stats.py:578-614): window term + weights.frame x per-frame terms.
    Returns (loss: float, [(d_mean, d_cov)] per frame)."""
    ref_mean, ref_cov = reference
    if window is not None:
        lo, hi = window
        profiles = profiles[lo:hi]
    if not profiles:
        raise ValueError("empty profile window")
    dev = _t(profiles[0][0]).device
    ref_mean, ref_cov = _t(ref_mean, dev), _t(ref_cov, dev)
    for m, cv in profiles:
        if tuple(m.shape) != tuple(ref_mean.shape) or \
                tuple(cv.shape) != tuple(ref_cov.shape):
            raise ValueError("profile and reference shapes differ")
    ny = ref_mean.shape[0]
    wm = torch.as_tensor(weights.mean, dtype=F64, device=dev)
    wc = torch.as_tensor(weights.cov, dtype=F64, device=dev)

    def term_grad(mean, cov, scale):
        dm = scale * wm[None, :] * 2.0 * (mean - ref_mean) / ny
        dc = scale * wc[None, :, :] * 2.0 * (cov - ref_cov) / ny
        return dm, dc

    win_mean, win_cov = window_profile(profiles)
    loss = _term(win_mean, win_cov, ref_mean, ref_cov, wm, wc)
    dwm, dwc = term_grad(win_mean, win_cov, 1.0)
    grads = window_profile_backward(profiles, dwm, dwc)
    for t, (m, cv) in enumerate(profiles):
        m, cv = _t(m, dev), _t(cv, dev)
        loss = loss + weights.frame * _term(m, cv, ref_mean, ref_cov, wm, wc)
        dm, dc = term_grad(m, cv, weights.frame)
        grads[t] = (grads[t][0] + dm, grads[t][1] + dc)
    return float(loss), grads


def stats_loss(profiles, reference, weights, window=None):
    """Weighted statistics loss over a rollout window (S/stats.py:567-575)."""
    return stats_loss_grad(profiles, reference, weights, window)[0]


def stats_loss_torch(profiles, reference, weights):
    """The same loss as a differentiable torch expression of the frame
    profiles (for FrameProfile outputs inside a training graph)."""
    ref_mean, ref_cov = reference
    dev = profiles[0][0].device
    ref_mean, ref_cov = _t(ref_mean, dev), _t(ref_cov, dev)
    wm = torch.as_tensor(weights.mean, dtype=F64, device=dev)
    wc = torch.as_tensor(weights.cov, dtype=F64, device=dev)
    means = torch.stack([m for m, _ in profiles])
    covs = torch.stack([c for _, c in profiles])
    mu = means.mean(dim=0)
    dv = means - mu
    wcov = covs.mean(dim=0) + torch.einsum("tyi,tyj->yij", dv, dv) / len(
        profiles)
    loss = _term(mu, wcov, ref_mean, ref_cov, wm, wc)
    for m, cv in profiles:
        loss = loss + weights.frame * _term(m, cv, ref_mean, ref_cov, wm, wc)
    return loss


# ---------------------------------------------------------------------------
# streaming statistics


@dataclass
class FrictionScales:
    u_tau: float
    re_tau: float
    delta: float
    nu: float

    def y_plus(self, dist_to_wall):
        return np.asarray(dist_to_wall) * self.u_tau / self.nu

    @property
    def t_plus_scale(self):
        return self.u_tau ** 2 / self.nu

    @property
    def ett_scale(self):
        return self.u_tau / self.delta


@dataclass
class StatsProfile:
    y: np.ndarray
    mean: np.ndarray                 # (Y, C)
    cov: np.ndarray                  # (Y, C, C)
    skewness: np.ndarray = None
    flatness: np.ndarray = None
    scales: FrictionScales = None
    y_walls: tuple = None

    @property
    def y_plus(self):
        if self.scales is None or self.y_walls is None:
            raise ValueError("profile carries no friction scaling")
        lo, hi = self.y_walls
        d_wall = np.minimum(self.y - lo, hi - self.y)
        return self.scales.y_plus(d_wall)


def friction_scales_from_profile(sl, u_mean, nu, wall_values=(0.0, 0.0)):
    """u_tau from one-sided slice-mean gradients at both walls, averaged
    (S/stats.py:417-425)."""
    u_mean = np.asarray(u_mean.detach().cpu() if torch.is_tensor(u_mean)
                        else u_mean)
    lo = abs((u_mean[0] - wall_values[0]) / (sl.y[0] - sl.y_lo))
    hi = abs((u_mean[-1] - wall_values[1]) / (sl.y_hi - sl.y[-1]))
    slope = 0.5 * (lo + hi)
    u_tau = float(np.sqrt(nu * slope))
    delta = sl.delta
    return FrictionScales(u_tau=u_tau, re_tau=u_tau * delta / nu,
                          delta=delta, nu=nu)


class ChannelAccumulator:
    """Per-slice moment accumulators fed frame by frame
    (S/stats.py:325-376): means, the full covariance and (``higher``) the
    third and fourth single-channel central moments.  Each frame's moments
    are formed on the device; frames merge with the exact pairwise update
    of central moment sums (Chan et al.), on the device."""

    def __init__(self, domain, wall_axis=1, higher=True):
        self.slices = channel_slices(domain, wall_axis)
        self.higher = higher
        self.time = 0.0
        self.count = 0.0
        self.mean = self.m2 = self.m3 = self.m4 = None

    def add_frame(self, u, dt=0.0):
        mean, cov, m3, m4 = frame_moments(self.slices, u, higher=True)
        nb = float(self.slices.m)
        self._merge(nb, mean, cov * nb, m3 * nb, m4 * nb)
        self.time += dt
        return self

    def _merge(self, nb, mean_b, m2b, m3b, m4b):
        if self.count == 0:
            self.count = nb
            self.mean, self.m2, self.m3, self.m4 = mean_b, m2b, m3b, m4b
            return
        na = self.count
        n = na + nb
        d = mean_b - self.mean                     # (Y, C)
        m2a, m3a, m4a = self.m2, self.m3, self.m4
        m2a_d = torch.diagonal(m2a, dim1=1, dim2=2)
        m2b_d = torch.diagonal(m2b, dim1=1, dim2=2)
        self.mean = self.mean + d * (nb / n)
        self.m2 = m2a + m2b + torch.einsum("yi,yj->yij", d, d) * (
            na * nb / n)
        self.m3 = (m3a + m3b + d ** 3 * (na * nb * (na - nb) / n ** 2)
                   + 3.0 * d * (na * m2b_d - nb * m2a_d) / n)
        self.m4 = (m4a + m4b
                   + d ** 4 * (na * nb * (na * na - na * nb + nb * nb)
                               / n ** 3)
                   + 6.0 * d ** 2 * (na * na * m2b_d + nb * nb * m2a_d)
                   / n ** 2
                   + 4.0 * d * (na * m3b - nb * m3a) / n)
        self.count = n

    def merge(self, other):
        out = ChannelAccumulator.__new__(ChannelAccumulator)
        out.slices, out.higher = self.slices, self.higher
        out.time = self.time + other.time
        out.count = self.count
        out.mean, out.m2, out.m3, out.m4 = self.mean, self.m2, self.m3, \
            self.m4
        if other.count:
            out._merge(other.count, other.mean, other.m2, other.m3, other.m4)
        return out

    def profile(self, nu=None):
        if not self.count:
            raise ValueError("empty accumulator has no mean")
        sl = self.slices
        mean = self.mean.detach().cpu().numpy()
        cov = (self.m2 / self.count).detach().cpu().numpy()
        skew = flat = None
        if self.higher:
            var = torch.diagonal(self.m2, dim1=1, dim2=2) / self.count
            m3 = self.m3 / self.count
            m4 = self.m4 / self.count
            pos = var > 0
            skew = torch.where(pos, m3 / var.clamp_min(1e-300) ** 1.5,
                               torch.zeros_like(m3)).cpu().numpy()
            flat = torch.where(pos, m4 / var.clamp_min(1e-300) ** 2,
                               torch.zeros_like(m4)).cpu().numpy()
        scales = None
        if nu is not None:
            scales = friction_scales_from_profile(sl, mean[:, 0], nu)
        return StatsProfile(y=sl.y.copy(), mean=mean, cov=cov,
                            skewness=skew, flatness=flat, scales=scales,
                            y_walls=(sl.y_lo, sl.y_hi))


__all__ = ["ChannelSlices", "channel_slices", "frame_moments",
           "frame_profile", "frame_profile_backward", "FrameProfile",
           "frame_profile_fn", "slice_mean", "slice_cov", "window_profile",
           "window_profile_backward", "LossWeights", "tcf_default_weights",
           "stats_loss", "stats_loss_grad", "stats_loss_torch",
           "FrictionScales", "StatsProfile", "friction_scales_from_profile",
           "ChannelAccumulator"]
