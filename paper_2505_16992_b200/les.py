"""Learned-SGS channel LES training step (BASELINE config 5).

The paper trains a CNN corrector S_theta(u) as a body force inside the PISO
step (the reference's hook is ``StepConfig.source``,
S/piso.py:50, with cotangent ``GradState.source``, S/adjoint.py:57).  One
training step here is:

1. a k-step unrolled rollout of the differentiable PISO step
   (:func:`~paper_2505_16992_b200.autograd.piso_step_fn`) on one
   64 x 48 x 64 channel sample per process, with source = wall forcing +
   S_theta(u);
2. a loss on the rollout: the paper's statistics loss (per-frame and
   window-averaged wall-normal mean / covariance profiles against reference
   statistics, S/stats.py:567-614, profiles from :mod:`.stats` on the
   device), or a plain mean-streamwise-profile loss;
3. ``loss.backward()`` -- the discrete adjoint through every step, then the
   CNN's own backward;
4. data-parallel gradient averaging across processes (one sample per GPU;
   the only collective of the path, SURVEY.md §8 e).

The CNN itself is an ordinary torch module (cuDNN convolutions); the PISO
step and its adjoint run in libpisob200.so.
"""

import torch
import torch.distributed as dist

from . import autograd as _ag


class SGSCorrector(torch.nn.Module):
    """Small 3D CNN mapping the velocity (n, 3) of a box grid to a body force
    (n, 3): periodic padding along the periodic axes, replicate along the
    walls."""

    def __init__(self, shape, periodic, width=8, scale=1e-3,
                 dtype=torch.float64):
        super().__init__()
        self.shape = tuple(shape)
        self.periodic = tuple(periodic)
        self.scale = scale
        # the corrector's own arithmetic type (float32 runs the convolutions
        # on the tensor cores); its input and output stay float64, the type
        # of the PISO step
        self.dtype = dtype
        self.c1 = torch.nn.Conv3d(3, width, 3, dtype=dtype)
        self.c2 = torch.nn.Conv3d(width, 3, 1, dtype=dtype)

    def _pad(self, x):
        out = x
        for ax in range(3):
            dim = 2 + ax
            if self.periodic[ax]:
                out = torch.cat([out.narrow(dim, out.shape[dim] - 1, 1), out,
                                 out.narrow(dim, 0, 1)], dim=dim)
            else:
                out = torch.cat([out.narrow(dim, 0, 1), out,
                                 out.narrow(dim, out.shape[dim] - 1, 1)],
                                dim=dim)
        return out

    def forward(self, u):
        x = u.t().reshape(1, 3, *self.shape).to(self.dtype)
        y = self.c2(torch.nn.functional.gelu(self.c1(self._pad(x))))
        return self.scale * y.reshape(3, -1).t().to(u.dtype)


def unrolled_loss(domain, u0, bc, model, forcing, nu, cfg, steps,
                  target_profile, step_fn=None):
    """Differentiable k-step rollout and its loss.  ``step_fn`` defaults to
    the PISO step (tests inject a CPU stand-in to exercise the host logic).
    Returns (loss, final velocity)."""
    step_fn = step_fn or (lambda u, src: _ag.piso_step_fn(domain, u, src, nu,
                                                          bc, cfg)[0])
    shape = model.shape
    u = u0
    loss = u0.new_zeros(())
    for _ in range(steps):
        src = forcing(u.detach(), nu) + model(u)
        u = step_fn(u, src)
        prof = u[:, 0].reshape(shape).mean(dim=(0, 2))
        loss = loss + ((prof - target_profile) ** 2).mean()
    return loss / steps, u


def stats_unrolled_loss(domain, u0, bc, model, forcing, nu, cfg, steps,
                        reference, weights, slices=None, step_fn=None):
    """Differentiable k-step rollout scored by the statistics loss of the
    training runs (S/stats.py:567-614): frame profiles from the device
    kernels (stats.FrameProfile), window + weighted per-frame terms.
    Returns (loss, final velocity)."""
    from . import stats as _st
    step_fn = step_fn or (lambda u, src: _ag.piso_step_fn(domain, u, src, nu,
                                                          bc, cfg)[0])
    sl = slices or _st.channel_slices(domain)
    u = u0
    profiles = []
    for _ in range(steps):
        src = forcing(u.detach(), nu) + model(u)
        u = step_fn(u, src)
        profiles.append(_st.frame_profile_fn(sl, u))
    return _st.stats_loss_torch(profiles, reference, weights), u


def average_gradients(model):
    """All-reduce-mean the parameter gradients over the default process
    group (the data-parallel collective of config 5)."""
    if not (dist.is_available() and dist.is_initialized()):
        return
    world = dist.get_world_size()
    if world == 1:
        return
    grads = [p.grad for p in model.parameters() if p.grad is not None]
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat)
    flat /= world
    off = 0
    for g in grads:
        g.copy_(flat[off:off + g.numel()].reshape(g.shape))
        off += g.numel()


def train_step(domain, u0, bc, model, opt, forcing, nu, cfg, steps,
               target_profile, step_fn=None, stats_target=None):
    """One data-parallel training step; returns the (local) loss value.
    ``stats_target`` = (reference (mean, cov), LossWeights[, slices])
    selects the statistics loss instead of the mean-profile loss."""
    opt.zero_grad(set_to_none=True)
    if stats_target is not None:
        ref, weights = stats_target[0], stats_target[1]
        sl = stats_target[2] if len(stats_target) > 2 else None
        loss, _ = stats_unrolled_loss(domain, u0, bc, model, forcing, nu,
                                      cfg, steps, ref, weights, sl, step_fn)
    else:
        loss, _ = unrolled_loss(domain, u0, bc, model, forcing, nu, cfg,
                                steps, target_profile, step_fn)
    loss.backward()
    average_gradients(model)
    opt.step()
    return float(loss.detach())


__all__ = ["SGSCorrector", "unrolled_loss", "stats_unrolled_loss",
           "average_gradients", "train_step"]
