"""``torch.autograd`` face of the differentiable PISO step.

``piso_step_fn(domain, u, source, nu, bc, cfg, ...)`` advances one step
with :func:`~paper_2505_16992_b200.piso.piso_step` and registers the
hand-written discrete adjoint (:func:`~paper_2505_16992_b200.adjoint.
backward_step`) as its backward, so a learned corrector S_theta(u) (the
paper's SGS model; the reference's ``StepConfig.source`` hook,
S/piso.py:50) can be trained with ``loss.backward()`` through unrolled
steps.  Gradients flow to the input velocity, the body force (per-cell
(n, d) or uniform (d,)), the viscosity and the boundary velocities; the
input pressure only seeds warm starts and gets no gradient (as in
S/adjoint.py:505).
"""

from dataclasses import replace

import torch

from . import adjoint as _adj
from . import piso as _piso


class _PisoStep(torch.autograd.Function):

    @staticmethod
    def forward(ctx, u, source, nu, bc, p, domain, cfg, workspace, path,
                adj_tol, adj_maxiter):
        plan = domain.device_plan(u.device)
        state = _piso.FlowState(
            u=u.detach(), p=p.detach(),
            bc=_piso.bc_views(plan, None if bc is None else
                              bc.detach().t().contiguous()),
            t=0.0, step=0)
        src = None if source is None else source.detach()
        cfg2 = replace(cfg, nu=float(nu), source=src)
        tape = _piso.StepTape()
        new, diag = _piso.piso_step(domain, state, cfg2, workspace, tape)
        ctx.domain, ctx.tape, ctx.path = domain, tape, path
        ctx.adj_tol, ctx.adj_maxiter = adj_tol, adj_maxiter
        ctx.src_shape = None if source is None else tuple(source.shape)
        ctx.has_bc = bc is not None
        ctx.diag = diag
        bc_out = (torch.cat([b for b in new.bc], 0) if new.bc
                  else torch.zeros((0, domain.dim), dtype=u.dtype,
                                   device=u.device))
        ctx.mark_non_differentiable(bc_out)
        return new.u, new.p, bc_out

    @staticmethod
    def backward(ctx, gu, gp, _gbc):
        if ctx.tape is None:
            raise RuntimeError(
                "piso_step_fn: the step's tape was released by an earlier "
                "backward pass; a second backward through the same step "
                "needs a fresh forward (retain_graph does not keep the "
                "device tape)")
        dom = ctx.domain
        dev = ctx.tape.c_data.device
        n, d = dom.n, dom.dim
        if gu is None:
            gu = torch.zeros((n, d), dtype=torch.float64, device=dev)
        g = _adj.backward_step(dom, ctx.tape, _adj.GradState(u=gu, p=gp),
                               path=ctx.path, tol=ctx.adj_tol,
                               maxiter=ctx.adj_maxiter)
        g_src = None
        if ctx.src_shape is not None:
            g_src = g.source if ctx.src_shape == (n, d) else \
                g.source.sum(dim=0)
        g_bc = torch.cat(list(g.bc), 0) if (ctx.has_bc and g.bc) else None
        g_nu = torch.tensor(g.nu, dtype=torch.float64, device=dev)
        ctx.tape = None
        return (g.u, g_src, g_nu, g_bc, None, None, None, None, None, None,
                None)


def piso_step_fn(domain, u, source, nu, bc, cfg, p=None, workspace=None,
                 path=_adj.GradientPath.FULL, adj_tol=None, adj_maxiter=None):
    """Differentiable PISO step.

    u: (n, d) velocity; source: None, (d,) or (n, d) body force; nu: float
    or 0-d tensor; bc: (m, d) boundary velocities (faces concatenated in
    ``domain.bfaces`` order) or None; cfg: StepConfig (its ``nu`` and
    ``source`` are overridden).  Returns (u_new, p_new, bc_new) with
    bc_new non-differentiable (the outflow update is not differentiated,
    S/piso.py:463-465).
    """
    if not torch.is_tensor(nu):
        nu = torch.tensor(float(nu), dtype=torch.float64, device=u.device)
    if p is None:
        p = torch.zeros(domain.n, dtype=torch.float64, device=u.device)
    if bc is None and domain.bfaces:
        raise ValueError("bc is required on domains with boundary faces")
    return _PisoStep.apply(u, source, nu, bc, p, domain, cfg, workspace,
                           path, adj_tol, adj_maxiter)


__all__ = ["piso_step_fn"]
