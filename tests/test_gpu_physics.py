"""GPU tier: physical and algebraic properties of the device step, the
reference's own physics battery (T/test_piso.py:22-137, T/test_linalg.py:
120-131) restated on the CUDA path: matrix structure, second-order
Poiseuille convergence on straight and distorted (non-orthogonal) meshes,
global conservation, projection, and the transpose-solve adjoint identity."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def _np(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def test_time_term_dominates_at_tiny_viscosity():
    from paper_2505_16992_b200 import mesh, piso
    dom = mesh.make_box((4, 4), periodic=(False, False))
    dt = 0.25
    c = _np(piso.assemble_momentum(dom, torch.zeros((dom.n, 2),
                                                    dtype=torch.float64,
                                                    device=DEV), 1e-30, dt))
    assert np.allclose(c[0], 1.0 / dt, rtol=1e-12)
    assert np.abs(c[1:]).max() < 1e-25


def test_constant_advection_row_sums_are_the_time_term():
    from paper_2505_16992_b200 import linalg, mesh, piso
    dom = mesh.make_box((6, 5))
    u = torch.tensor([0.7, -0.3], dtype=torch.float64,
                     device=DEV).repeat(dom.n, 1)
    dt = 0.1
    c = piso.assemble_momentum(dom, u, 0.05, dt)
    rows = linalg.stencil_to_csr(dom, c) @ np.ones(dom.n)
    assert np.allclose(rows, 1.0 / dt, atol=1e-13)


def test_pressure_matrix_symmetric_zero_rowsums_negative_diagonal():
    from paper_2505_16992_b200 import linalg, mesh, piso
    dom = mesh.make_poiseuille((8, 6), distort=0.25)
    rng = np.random.default_rng(0)
    a_inv = torch.as_tensor(0.5 + rng.random(dom.n), device=DEV)
    p = piso.assemble_pressure(dom, a_inv)
    csr = linalg.stencil_to_csr(dom, p)
    assert abs(csr - csr.T).max() == 0.0
    rows = csr @ np.ones(dom.n)
    assert np.abs(rows).max() < 1e-14 * np.abs(csr.data).max()
    assert (_np(p)[0] < 0).all()


def _poiseuille_error(ny, distort=0.0, nonortho=0, steps=90):
    from paper_2505_16992_b200 import mesh, piso
    dom = mesh.make_poiseuille((4 if not distort else 24, ny),
                               distort=distort)
    cfg = piso.StepConfig(dt=0.05, nu=1.0, source=(1.0, 0.0), tol=1e-10,
                          nonortho_correctors=nonortho)
    st = piso.make_state(dom, device=DEV)
    ws = piso.PisoWorkspace(dom)
    for _ in range(steps):
        st, diag = piso.piso_step(dom, st, cfg, ws)
    y = dom.centers[:, 1]
    exact = 0.5 * y * (1.0 - y)
    u = _np(st.u)
    return np.abs(u[:, 0] - exact).max() / exact.max(), u


def test_poiseuille_converges_to_parabola_second_order():
    err32, u = _poiseuille_error(32)
    assert err32 < 0.02
    assert np.abs(u[:, 1]).max() < 1e-8
    errs = [_poiseuille_error(ny)[0] for ny in (8, 16, 32)]
    assert errs[0] > errs[1] > errs[2]
    assert errs[1] / errs[2] > 3.0


def test_poiseuille_distorted_mesh_nonortho_correctors():
    err, u = _poiseuille_error(24, distort=0.3, nonortho=2, steps=120)
    assert err < 0.06
    assert np.isfinite(u).all()


@pytest.mark.parametrize("case", ["cavity", "rotated_two_block"])
def test_global_conservation(case):
    from paper_2505_16992_b200 import mesh, piso
    rng = np.random.default_rng(3)
    if case == "cavity":
        dom = mesh.make_cavity((8, 8))
        st = piso.make_state(dom, u0=rng.standard_normal((dom.n, 2)) * 0.1,
                             device=DEV)
        b = piso.divergence_rhs(dom, st.u, st.bc)
        assert abs(float(b.sum())) < 1e-13
    else:
        dom = mesh.make_two_block((6, 6), rotated=True)
        u = torch.as_tensor(rng.standard_normal((dom.n, 2)), device=DEV)
        bc = [np.zeros((f.m, 2)) for f in dom.bfaces]
        b = piso.divergence_rhs(dom, u, bc)
        assert abs(float(b.sum())) < 1e-12


def test_projection_reduces_divergence():
    from paper_2505_16992_b200 import mesh, piso
    dom = mesh.make_box((16, 16))
    x, y = dom.centers[:, 0], dom.centers[:, 1]
    u0 = 0.1 * np.stack([np.sin(2 * np.pi * x / 16),
                         np.sin(2 * np.pi * y / 16)], axis=-1)
    st = piso.make_state(dom, u0=u0, device=DEV)
    div0 = float(piso.divergence(dom, st.u, st.bc).abs().max())
    cfg = piso.StepConfig(dt=0.02, nu=0.05, tol=1e-11)
    new, diag = piso.piso_step(dom, st, cfg)
    assert diag.div_contract < 10 * 1e-11
    div1 = float(piso.divergence(dom, new.u, new.bc).abs().max())
    assert div1 < 0.1 * div0


@pytest.mark.parametrize("shape", [(12, 10), (8, 16, 32)])
def test_transpose_solve_adjoint_identity(shape):
    """<A^-1 b, c> = <b, A^-t c> through the forward and transposed
    BiCGStab (the identity the discrete adjoint rests on)."""
    from paper_2505_16992_b200 import channel, linalg, mesh, piso
    dom = (mesh.make_cavity(shape) if len(shape) == 2
           else mesh.make_channel(shape, ratio=1.1))
    if dom.dim == 3:
        u, nu, _ = channel.reichardt_velocity(dom, 180.0, device=DEV)
    else:
        rng = np.random.default_rng(1)
        u = torch.as_tensor(0.3 * rng.standard_normal((dom.n, 2)),
                            device=DEV)
        nu = 0.01
    c = piso.assemble_momentum(dom, u, nu, 0.01)
    plan = dom.device_plan(DEV)
    g = torch.Generator(device="cpu").manual_seed(2)
    b = torch.randn(dom.n, generator=g, dtype=torch.float64).to(DEV)
    w = torch.randn(dom.n, generator=g, dtype=torch.float64).to(DEV)
    x, _ = linalg.bicgstab_solve(plan, c, b, tol=1e-13)
    y, _ = linalg.bicgstab_solve(plan, c, w, tol=1e-13, transpose=True)
    lhs, rhs = float((x * w).sum()), float((b * y).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs))
