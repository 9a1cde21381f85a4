"""GPU tier: the channel drivers on the device (S/piso.py:
512-546, 668-714) -- reichardt_init, the fused wall-forcing kernel and
adaptive_dt's CFL-peak kernel -- against the reference's golden vectors
(tests/golden/reichardt.npz) and the reference itself run live
(oracle/_ref)."""

import numpy as np
import pytest
import torch

import golden_cases as G
import ref_live as RL

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("tag", ["a", "b"])
def test_reichardt_and_forcing_on_device_match_golden(tag):
    from paper_2505_16992_b200 import channel, mesh
    g = G.load("reichardt")
    dom = mesh.make_channel(tuple(g[f"{tag}_shape"]),
                            ratio=float(g[f"{tag}_ratio"]))
    u, nu, ut = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=3, device=DEV)
    assert u.is_cuda
    assert nu == pytest.approx(float(g[f"{tag}_nu"]), rel=1e-15)
    assert ut == pytest.approx(float(g[f"{tag}_utau"]), rel=1e-15)
    assert G.rel(u.cpu().numpy(), g[f"{tag}_u"]) < 1e-13
    f = channel.WallForcing(dom, DEV)(u, nu)
    assert f.is_cuda
    assert G.rel(f.cpu().numpy(), g[f"{tag}_forcing"]) < 1e-12
    f2 = channel.wall_forcing_source(dom, u, nu)
    assert torch.equal(f, f2)


@pytest.fixture(scope="module")
def R():
    r = RL.reference()
    if r is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    return r


@pytest.mark.parametrize("case", ["channel", "cavity", "obstacle"])
def test_adaptive_dt_and_forcing_match_reference(R, case):
    from paper_2505_16992_b200 import channel, mesh
    RM, RP = R["mesh"], R["piso"]
    rng = np.random.default_rng(4)
    if case == "channel":
        rd = RM.make_channel((8, 16, 32), ratio=1.1)
        dom = mesh.make_channel((8, 16, 32), ratio=1.1)
    elif case == "cavity":
        rd, dom = RM.make_cavity((12, 9)), mesh.make_cavity((12, 9))
    else:
        rd, dom = RL.obstacle(RM, q=4), RL.obstacle(mesh, q=4)
    u = rng.standard_normal((dom.n, dom.dim))
    ut = torch.as_tensor(u, device=DEV)
    for cfl, dtmax, rem in [(0.5, 1.0, None), (0.3, 1e-4, None),
                            (0.8, 1.0, 1e-3)]:
        ours = channel.adaptive_dt(dom, ut, cfl, dtmax, rem)
        ref = RP.adaptive_dt(rd, u, cfl, dtmax, rem)
        assert ours == pytest.approx(ref, rel=1e-14), (cfl, ours, ref)
    zero = torch.zeros_like(ut)
    assert channel.adaptive_dt(dom, zero, 0.5, 0.25) == 0.25
    if case != "cavity":
        return
    # the cavity's Dirichlet walls along axis 1 (the lid moves: u/dist of
    # its first row enters the mean like any wall's)
    nu = 0.0123
    ours = channel.wall_forcing_source(dom, ut, nu).cpu().numpy()
    ref = RP.wall_forcing_source(rd, u, nu)
    assert RL.rel(ours, ref) < 1e-13
