"""GPU tier: the torch.autograd wrapper reproduces backward_step and
trains a learned body force through unrolled steps (FD-checked)."""

import numpy as np
import pytest
import torch

import golden_cases as G

pytestmark = pytest.mark.gpu


def test_autograd_matches_backward_step():
    from paper_2505_16992_b200 import adjoint, autograd, piso
    g = G.load("cavity8")
    dom = G.build("cavity8")
    dev = torch.device("cuda:0")
    u0 = torch.as_tensor(g["u0"], device=dev).requires_grad_(True)
    src = torch.as_tensor(np.random.default_rng(1).standard_normal(
        (dom.n, 2)) * 0.1, device=dev).requires_grad_(True)
    bc = torch.as_tensor(g["bc0"], device=dev).requires_grad_(True)
    nu = torch.tensor(float(g["nu"]), dtype=torch.float64, device=dev,
                      requires_grad=True)
    cfg = piso.StepConfig(dt=float(g["dt"]), nu=float(g["nu"]), tol=1e-12)
    u1, p1, _ = autograd.piso_step_fn(dom, u0, src, nu, bc, cfg,
                                      adj_tol=1e-12)
    wu = torch.as_tensor(g["cot_u"], device=dev)
    wp = torch.as_tensor(g["cot_p"], device=dev)
    loss = (u1 * wu).sum() + (p1 * wp).sum()
    loss.backward()
    # direct adjoint on the same inputs
    st = piso.make_state(dom, u0=g["u0"], device=dev)
    for b, ref in zip(st.bc, G.split_bc(g, g["bc0"])):
        b.copy_(torch.as_tensor(ref, device=dev))
    tape = piso.StepTape()
    piso.piso_step(dom, st, piso.StepConfig(dt=cfg.dt, nu=cfg.nu,
                                            source=src.detach(), tol=1e-12),
                   tape=tape)
    gd = adjoint.backward_step(dom, tape, adjoint.GradState(u=wu, p=wp),
                               tol=1e-12)
    assert torch.allclose(u0.grad, gd.u, rtol=0, atol=1e-14)
    assert torch.allclose(src.grad, gd.source, rtol=0, atol=1e-14)
    assert float(nu.grad) == pytest.approx(gd.nu, rel=1e-14)
    assert torch.allclose(bc.grad, torch.cat(list(gd.bc), 0), atol=1e-14)


def test_unrolled_learned_source_gradient_fd():
    """S_theta(u) = theta * u (a stand-in corrector) through 3 steps; the
    gradient w.r.t. theta agrees with central finite differences."""
    from paper_2505_16992_b200 import autograd, mesh, piso
    dom = mesh.make_box((6, 5, 4))
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(2)
    u0 = torch.as_tensor(0.3 * rng.standard_normal((dom.n, 3)), device=dev)
    w = torch.as_tensor(rng.standard_normal((dom.n, 3)), device=dev)
    cfg = piso.StepConfig(dt=0.1, nu=0.2, tol=1e-13)

    def loss_of(theta):
        u = u0
        for _ in range(3):
            u, p, _ = autograd.piso_step_fn(dom, u, theta * u, cfg.nu, None,
                                            cfg, adj_tol=1e-13)
        return (u * w).sum()

    th = torch.tensor(0.7, dtype=torch.float64, device=dev,
                      requires_grad=True)
    loss = loss_of(th)
    loss.backward()
    eps = 1e-5
    with torch.no_grad():
        fd = (loss_of(torch.tensor(0.7 + eps, dtype=torch.float64,
                                   device=dev))
              - loss_of(torch.tensor(0.7 - eps, dtype=torch.float64,
                                     device=dev))) / (2 * eps)
    assert float(th.grad) == pytest.approx(float(fd), rel=1e-6)
