"""GPU tier: the BASELINE configurations at their FULL sizes (C2 wall-refined
1024^2 cavity, C3 8-block 2048x512 obstacle grid, C4 256x192x256 channel),
checked through size-independent properties, since the CPU oracle cannot
run them in test time:

* every linear solve converges and verifies its true residual (a
  non-converged solve raises SolverError with the reference's stage label);
* the projected velocity is discretely divergence-free to solver tolerance;
* the discrete adjoint is the exact transpose of the step's linearisation:
  the directional derivative of J(u0) = <w, u1> along a random v by central
  differences equals <dJ/du0, v> from backward_step (FULL path);
* the adjoint of nu: dJ/dnu against central differences.

Small-size parity against the reference's own golden vectors is in
test_gpu_parity.py; this file proves the same step at the benchmark sizes.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _c2():
    from paper_2505_16992_b200 import mesh
    dom = mesh.make_wall_refined_cavity(1024, ratio=1.0045)
    x = mesh.wall_refined_coords(1024, 0.5, 1.0045)
    dt = 25.0 * float(np.diff(x).min())
    return dom, 1e-3, dt, None


def _c3():
    from paper_2505_16992_b200 import mesh

    def inlet(fc):
        return np.stack([np.ones(len(fc)), np.zeros(len(fc))], axis=-1)
    dom = mesh.make_obstacle_grid(domain_size=(32.0, 8.0),
                                  obstacle_center=(6.5, 4.0),
                                  obstacle_size=(1.0, 1.0),
                                  nx=(384, 64, 1600), ny=(224, 64, 224),
                                  inlet=inlet)
    return dom, 0.01, 0.0125, None


def _c4():
    from paper_2505_16992_b200 import mesh
    dom = mesh.make_channel((256, 192, 256), ratio=1.03)
    return dom, None, None, (1e-3, 0.0, 0.0)


def _u0(dom, dev, seed):
    from paper_2505_16992_b200 import channel
    if dom.dim == 3:
        u, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                              seed=seed, device=dev)
        return u, nu
    g = torch.Generator(device="cpu").manual_seed(seed)
    u = 0.1 * torch.randn((dom.n, dom.dim), generator=g, dtype=torch.float64)
    return u.to(dev), None


@pytest.mark.parametrize("case", ["c2", "c3", "c4"])
def test_full_size_step_properties(case):
    from paper_2505_16992_b200 import adjoint, piso
    dev = torch.device("cuda:0")
    dom, nu, dt, src = {"c2": _c2, "c3": _c3, "c4": _c4}[case]()
    u0, nu_ch = _u0(dom, dev, 0)
    nu = nu if nu is not None else nu_ch
    if dt is None:
        dt = 0.3 * (2 * np.pi / 256) / float(u0.abs().max())
    d, n = dom.dim, dom.n
    g = torch.Generator(device="cpu").manual_seed(1)
    w = torch.randn((n, d), generator=g, dtype=torch.float64).to(dev)
    v = torch.randn((n, d), generator=g, dtype=torch.float64).to(dev)
    # the advective outflow update (S/piso.py:467-509) sits OUTSIDE the
    # differentiated step: keep the perturbation off the cells it reads
    for f in dom.bfaces:
        if f.kind == "advective_outflow":
            v[torch.as_tensor(f.cells, device=dev)] = 0.0
    base = piso.make_state(dom, u0=u0, device=dev)

    def J(u_init, nu_val, tape=None):
        st = piso.make_state(dom, u0=u_init, device=dev)
        for b, b0 in zip(st.bc, base.bc):
            b.copy_(b0)
        cfg = piso.StepConfig(dt=dt, nu=nu_val, source=src, tol=TOL)
        new, diag = piso.piso_step(dom, st, cfg, None, tape)
        return float((new.u * w).sum()), new, diag

    tape = piso.StepTape()
    j0, new, diag = J(u0, nu, tape)
    # every solve converged and verified (reports carry the true residual)
    for r in diag.reports:
        assert r.converged and r.residual <= 10 * TOL, r
    # projected velocity discretely divergence-free (contract residual of
    # the last pressure solve, relative to its rhs)
    assert diag.div_contract <= 10 * TOL
    gr = adjoint.backward_step(dom, tape, adjoint.GradState(
        u=w, p=torch.zeros(n, dtype=torch.float64, device=dev)), tol=TOL)
    an = float((gr.u * v).sum())
    # central differences: truncation O(eps^2) vs. the Krylov solves' own
    # tolerance noise (~TOL |J| / eps) -- a 1e-3 relative step balances them
    eps = 1e-3 * float(u0.abs().max()) / float(v.abs().max())
    jp, _, _ = J(u0 + eps * v, nu)
    jm, _, _ = J(u0 - eps * v, nu)
    fd = (jp - jm) / (2 * eps)
    assert abs(fd - an) <= 1e-5 * max(abs(an), abs(fd)), (case, fd, an)
    h = 1e-4 * nu
    fd_nu = (J(u0, nu + h)[0] - J(u0, nu - h)[0]) / (2 * h)
    assert abs(fd_nu - gr.nu) <= 1e-5 * max(abs(gr.nu), abs(fd_nu)), \
        (case, fd_nu, gr.nu)
