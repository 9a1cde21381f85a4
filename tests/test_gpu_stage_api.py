"""GPU tier: the reference's stage API on the device -- the exact transpose
identities of /root/reference/pkg/tests/test_adjoint.py:72-146 (restated for
this package's torch device tensors) and, where the reference builds here
(oracle/_ref), the same building blocks compared value for value with the
reference's own (S/piso.py:128-264, 322-342, 431-455; S/adjoint.py:78-205).
"""

import numpy as np
import pytest
import torch

import ref_live as RL

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _t(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=DEV)


def _n(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def _identity_domains(M):
    return [M.make_poiseuille((5, 4), distort=0.35),
            M.make_two_block((3, 3), rotated=True)]


def _close(lhs, rhs):
    return abs(lhs - rhs) < 1e-9 * max(1.0, abs(lhs))


def test_wide_grad_adjoint_identity():
    from paper_2505_16992_b200 import mesh, piso
    rng = np.random.default_rng(0)
    for dom in _identity_domains(mesh):
        phi = _t(rng.standard_normal(dom.n))
        for variant in ("mirror", "onesided"):
            cot = _t(rng.standard_normal((dom.n, dom.dim)))
            lhs = float((piso.wide_grad(dom, phi, variant) * cot).sum())
            rhs = float((phi * piso.wide_grad_adjoint(dom, cot, variant)).sum())
            assert _close(lhs, rhs), (variant, lhs, rhs)


def test_wide_grad_face_variant_adjoint_identity():
    from paper_2505_16992_b200 import mesh, piso
    rng = np.random.default_rng(1)
    dom = mesh.make_cavity((4, 5))
    phi = _t(rng.standard_normal(dom.n))
    bc_cells = {(a, s): _t(rng.standard_normal(dom.n))
                for a in range(2) for s in (0, 1)}
    cot = _t(rng.standard_normal((dom.n, 2)))
    lhs = float((piso.wide_grad(dom, phi, "face", bc_cells) * cot).sum())
    out, bc_cot = piso.wide_grad_adjoint(dom, cot, "face")
    rhs = float((phi * out).sum()) + sum(
        float((bc_cells[k] * bc_cot[k]).sum()) for k in bc_cells)
    assert _close(lhs, rhs)


def test_divergence_rhs_adjoint_identity():
    from paper_2505_16992_b200 import adjoint, mesh, piso
    rng = np.random.default_rng(2)
    for dom in _identity_domains(mesh):
        h = _t(rng.standard_normal((dom.n, dom.dim)))
        bc = [_t(rng.standard_normal((f.m, dom.dim))) for f in dom.bfaces]
        cot = _t(rng.standard_normal(dom.n))
        lhs = float((piso.divergence_rhs(dom, h, bc) * cot).sum())
        dh, dbc = adjoint._adj_divergence_rhs(dom, cot)
        rh = float((h * dh).sum())
        rb = sum(float((b * g).sum()) for b, g in zip(bc, dbc))
        assert _close(lhs, rh + rb), (dom.n, lhs, rh, rb)


def test_momentum_cross_adjoint_identity():
    from paper_2505_16992_b200 import adjoint, mesh, piso
    rng = np.random.default_rng(3)
    for dom in _identity_domains(mesh):
        u = _t(rng.standard_normal((dom.n, dom.dim)))
        cot = _t(rng.standard_normal((dom.n, dom.dim)))
        nu = 0.37
        lhs = float((piso.momentum_cross_rhs(dom, u, nu) * cot).sum())
        du, dnu = adjoint._adj_momentum_cross(dom, u, nu, cot)
        assert _close(lhs, float((u * du).sum()))
        # linear in nu: nu * dnu recovers the value
        assert _close(lhs, nu * dnu)


def test_pressure_cross_adjoint_identity():
    from paper_2505_16992_b200 import adjoint, mesh, piso
    rng = np.random.default_rng(4)
    dom = mesh.make_poiseuille((5, 4), distort=0.35)
    p = _t(rng.standard_normal(dom.n))
    a_inv = _t(0.5 + rng.random(dom.n))
    cot = _t(rng.standard_normal(dom.n))
    lhs = float((piso.pressure_cross_rhs(dom, a_inv, p) * cot).sum())
    dp, d_ainv = adjoint._adj_pressure_cross(dom, a_inv, p, cot)
    assert _close(float((p * dp).sum()), lhs)
    assert _close(float((a_inv * d_ainv).sum()), lhs)


def test_correct_velocity_adjoint_identity():
    from paper_2505_16992_b200 import adjoint, mesh, piso
    rng = np.random.default_rng(5)
    dom = mesh.make_two_block((3, 3), rotated=True)
    h = _t(rng.standard_normal((dom.n, 2)))
    p = _t(rng.standard_normal(dom.n))
    a_diag = _t(1.0 + rng.random(dom.n))
    cot = _t(rng.standard_normal((dom.n, 2)))
    lhs = float((piso.correct_velocity(dom, h, p, 1.0 / a_diag) * cot).sum())
    dA, dp, dh = adjoint.backward_correct_velocity(dom, p, a_diag, cot)
    rhs = float((h * dh).sum()) + float((p * dp).sum())
    assert _close(lhs, rhs)


# ---------------------------------------------------------------------------
# value for value against the reference's own building blocks


@pytest.fixture(scope="module")
def R():
    r = RL.reference()
    if r is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    return r


def _pair(R, build):
    from paper_2505_16992_b200 import mesh
    return build(R["mesh"]), build(mesh)


BUILDS = [lambda M: M.make_poiseuille((5, 4), distort=0.35),
          lambda M: M.make_two_block((3, 3), rotated=True),
          lambda M: M.make_cavity((4, 5)),
          lambda M: M.make_channel((6, 8, 4), ratio=1.1)]


@pytest.mark.parametrize("k", range(len(BUILDS)))
def test_building_blocks_match_reference(R, k):
    from paper_2505_16992_b200 import adjoint, piso
    rdom, dom = _pair(R, BUILDS[k])
    RP, RA = R["piso"], R["adjoint"]
    rng = np.random.default_rng(10 + k)
    n, d = dom.n, dom.dim
    phi = rng.standard_normal(n)
    u = rng.standard_normal((n, d))
    cot = rng.standard_normal((n, d))
    cots = rng.standard_normal(n)
    a_diag = 1.0 + rng.random(n)
    worst = {}

    def chk(name, ours, ref, tol=1e-12):
        e = RL.rel(_n(ours), ref)
        worst[name] = e
        assert e < tol, (name, e)

    for variant in ("mirror", "onesided"):
        chk(f"wide_grad[{variant}]", piso.wide_grad(dom, _t(phi), variant),
            RP.wide_grad(rdom, phi, variant))
        chk(f"wide_grad_adjoint[{variant}]",
            piso.wide_grad_adjoint(dom, _t(cot), variant),
            RP.wide_grad_adjoint(rdom, cot, variant))
    chk("wide_grad[vector]", piso.wide_grad(dom, _t(u), "onesided"),
        RP.wide_grad(rdom, u, "onesided"))
    chk("momentum_cross_rhs", piso.momentum_cross_rhs(dom, _t(u), 0.37),
        RP.momentum_cross_rhs(rdom, u, 0.37))
    chk("pressure_cross_rhs",
        piso.pressure_cross_rhs(dom, _t(1.0 / a_diag), _t(phi)),
        RP.pressure_cross_rhs(rdom, 1.0 / a_diag, phi))
    chk("correct_velocity",
        piso.correct_velocity(dom, _t(u), _t(phi), _t(1.0 / a_diag)),
        RP.correct_velocity(rdom, u, phi, 1.0 / a_diag))
    dA, dp, dh = adjoint.backward_correct_velocity(dom, _t(phi), _t(a_diag),
                                                   _t(cot))
    rA, rp, rh = RA.backward_correct_velocity(rdom, phi, a_diag, cot)
    chk("backward_correct_velocity.dA", dA, rA)
    chk("backward_correct_velocity.dp", dp, rp)
    chk("backward_correct_velocity.dh", dh, rh)
    dh2, dbc = adjoint._adj_divergence_rhs(dom, _t(cots))
    rh2, rbc = RA._adj_divergence_rhs(rdom, cots)
    chk("_adj_divergence_rhs.dh", dh2, rh2)
    if rbc:
        chk("_adj_divergence_rhs.dbc", np.concatenate([_n(b) for b in dbc]),
            np.concatenate(rbc))
    if RP._has_cross_terms(rdom):
        du, dnu = adjoint._adj_momentum_cross(dom, _t(u), 0.37, _t(cot))
        rdu, rdnu = RA._adj_momentum_cross(rdom, u, 0.37, cot)
        chk("_adj_momentum_cross.du", du, rdu)
        assert abs(dnu - rdnu) <= 1e-12 * max(1.0, abs(rdnu))
        dpp, dai = adjoint._adj_pressure_cross(dom, _t(1.0 / a_diag),
                                               _t(phi), _t(cots))
        rdpp, rdai = RA._adj_pressure_cross(rdom, 1.0 / a_diag, phi, cots)
        chk("_adj_pressure_cross.dp", dpp, rdpp)
        chk("_adj_pressure_cross.d_ainv", dai, rdai)
    print(f"\n[stage API case {k}] worst rel. error: "
          + ", ".join(f"{kk}={v:.1e}" for kk, v in worst.items()))
