"""GPU tier: finite-difference gradchecks of whole steps and rollouts through
the device path, with the reference's harness semantics and thresholds
(T/test_adjoint.py:241-329 restated against this package)."""

from dataclasses import replace

import numpy as np
import pytest
import torch

from paper_2505_16992_b200 import mesh
from paper_2505_16992_b200.adjoint import (GradientPath, GradState,
                                           backward_rollout, gradcheck)
from paper_2505_16992_b200.piso import StepConfig, StepTape, make_state, \
    piso_step

pytestmark = pytest.mark.gpu
TIGHT = 1e-13
DEV = "cuda:0"


def loss_fn(domain, cfg, wu, wp, steps=1, lid_face=None, lid_profile=None):
    wu_t = torch.as_tensor(wu, device=DEV)
    wp_t = torch.as_tensor(wp, device=DEV)

    def fn(inp):
        c = replace(cfg, nu=float(inp["nu"]),
                    source=np.asarray(inp["src"], dtype=np.float64))
        state = make_state(domain, u0=np.asarray(inp["u0"]), device=DEV)
        if lid_face is not None:
            state.bc[lid_face].copy_(torch.as_tensor(
                float(inp["lid"]) * lid_profile, device=DEV))
        tapes = []
        for _ in range(steps):
            t = StepTape()
            state, _ = piso_step(domain, state, c, tape=t)
            tapes.append(t)
        loss = float((wu_t * state.u).sum() + (wp_t * state.p).sum())
        cots = [None] * (steps - 1) + [GradState(u=wu_t, p=wp_t)]
        g = backward_rollout(domain, tapes, cots, path=GradientPath.FULL,
                             tol=1e-12)
        grads = {"u0": g.u.cpu().numpy(), "nu": g.nu,
                 "src": g.source.cpu().numpy()}
        if lid_face is not None:
            grads["lid"] = float(np.vdot(g.bc[lid_face].cpu().numpy(),
                                         lid_profile))
        return loss, grads

    return fn


def test_gradcheck_step_cavity_all_inputs():
    dom = mesh.make_cavity((5, 5))
    rng = np.random.default_rng(9)
    lid = next(i for i, f in enumerate(dom.bfaces)
               if f.axis == 1 and f.side == 0)
    profile = np.stack([np.ones(dom.bfaces[lid].m),
                        np.zeros(dom.bfaces[lid].m)], axis=-1)
    cfg = StepConfig(dt=0.08, nu=0.15, tol=TIGHT)
    fn = loss_fn(dom, cfg, rng.standard_normal((dom.n, 2)),
                 rng.standard_normal(dom.n), lid_face=lid,
                 lid_profile=profile)
    inputs = {"u0": 0.2 * rng.standard_normal((dom.n, 2)), "nu": 0.15,
              "src": 0.1 * rng.standard_normal((dom.n, 2)), "lid": 0.8}
    rep = gradcheck(fn, inputs, stage="step_cavity")
    assert rep.passed, rep.text()


def test_gradcheck_step_distorted_nonortho():
    dom = mesh.make_poiseuille((6, 4), distort=0.35)
    rng = np.random.default_rng(10)
    cfg = StepConfig(dt=0.07, nu=0.2, nonortho_correctors=2, tol=TIGHT)
    fn = loss_fn(dom, cfg, rng.standard_normal((dom.n, 2)),
                 rng.standard_normal(dom.n))
    inputs = {"u0": 0.3 * rng.standard_normal((dom.n, 2)), "nu": 0.2,
              "src": np.zeros((dom.n, 2))}
    rep = gradcheck(fn, inputs, stage="step_nonortho")
    assert rep.passed, rep.text()


def test_gradcheck_step_rotated_two_block():
    dom = mesh.make_two_block((3, 3), rotated=True)
    rng = np.random.default_rng(11)
    cfg = StepConfig(dt=0.09, nu=0.3, tol=TIGHT)
    fn = loss_fn(dom, cfg, rng.standard_normal((dom.n, 2)),
                 rng.standard_normal(dom.n))
    inputs = {"u0": 0.25 * rng.standard_normal((dom.n, 2)), "nu": 0.3,
              "src": np.zeros((dom.n, 2))}
    rep = gradcheck(fn, inputs, stage="step_two_block")
    assert rep.passed, rep.text()


def test_gradcheck_step_3d_box():
    dom = mesh.make_box((4, 4, 4))
    rng = np.random.default_rng(12)
    cfg = StepConfig(dt=0.1, nu=0.25, tol=TIGHT)
    fn = loss_fn(dom, cfg, rng.standard_normal((dom.n, 3)),
                 rng.standard_normal(dom.n))
    inputs = {"u0": 0.2 * rng.standard_normal((dom.n, 3)), "nu": 0.25,
              "src": np.zeros((dom.n, 3))}
    rep = gradcheck(fn, inputs, stage="step_3d")
    assert rep.passed, rep.text()


def test_gradcheck_rollout_three_steps_channel_multigrid():
    """Wall-refined channel: the pressure solves run the multigrid PCG."""
    dom = mesh.make_channel((4, 6, 4), ratio=1.2)
    assert dom.device_plan(DEV).has_mg
    rng = np.random.default_rng(13)
    cfg = StepConfig(dt=0.06, nu=0.2, tol=TIGHT)
    fn = loss_fn(dom, cfg, rng.standard_normal((dom.n, 3)),
                 rng.standard_normal(dom.n), steps=3)
    inputs = {"u0": 0.2 * rng.standard_normal((dom.n, 3)), "nu": 0.2,
              "src": 0.05 * rng.standard_normal((dom.n, 3))}
    rep = gradcheck(fn, inputs, stage="rollout3")
    assert rep.passed, rep.text()


def test_gradcheck_negative_control():
    dom = mesh.make_cavity((4, 4))
    rng = np.random.default_rng(14)
    cfg = StepConfig(dt=0.08, nu=0.2, tol=TIGHT)
    clean = loss_fn(dom, cfg, rng.standard_normal((dom.n, 2)),
                    np.zeros(dom.n))

    def corrupted(inp):
        loss, grads = clean(inp)
        grads["u0"] = grads["u0"] * 1.01
        return loss, grads

    inputs = {"u0": 0.2 * rng.standard_normal((dom.n, 2)), "nu": 0.2,
              "src": np.zeros((dom.n, 2))}
    rep = gradcheck(corrupted, inputs, stage="negative")
    assert not rep.passed
    assert "u0" in {e.name for e in rep.entries if not e.passed}


def test_gradient_paths_structure():
    """T/test_adjoint.py:360-384: NONE skips every transpose solve, FULL
    costs the most, each gate changes the gradient, increments telescope."""
    from paper_2505_16992_b200.adjoint import backward_step
    dom = mesh.make_cavity((6, 6))
    rng = np.random.default_rng(15)
    cfg = StepConfig(dt=0.08, nu=0.15, tol=TIGHT)
    st = make_state(dom, u0=0.3 * rng.standard_normal((dom.n, 2)),
                    device=DEV)
    tape = StepTape()
    piso_step(dom, st, cfg, tape=tape)
    wu = torch.as_tensor(rng.standard_normal((dom.n, 2)), device=DEV)
    g = {p: backward_step(dom, tape, GradState(u=wu, p=None), path=p,
                          tol=1e-12) for p in GradientPath}
    full, none = g[GradientPath.FULL], g[GradientPath.NONE]
    adv, pon = g[GradientPath.ADV_ONLY], g[GradientPath.P_ONLY]
    assert none.solve_iterations == 0
    assert float(none.u.abs().max()) > 0
    assert full.solve_iterations > max(adv.solve_iterations,
                                       pon.solve_iterations)
    assert float((full.u - none.u).abs().max()) > 1e-8
    assert float((full.u - adv.u).abs().max()) > 1e-10
    assert float((full.u - pon.u).abs().max()) > 1e-10
