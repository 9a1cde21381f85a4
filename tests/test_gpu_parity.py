"""GPU tier: the CUDA path (through libpisob200.so) against the reference's
golden vectors and the CPU oracle on identical inputs and tolerances."""

import numpy as np
import pytest
import torch

import golden_cases as G
from oracle import pisoref as O

pytestmark = pytest.mark.gpu

GPU_TOL = 1e-12       # solver tolerance on the device
FIELD_TOL = 1e-8      # relative L-inf parity (north star asks 1e-6 in fp64)


def _np(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def _gpu_rollout(name, tol=GPU_TOL):
    from paper_2505_16992_b200 import piso
    g = G.load(name)
    dom = G.build(name)
    dev = torch.device("cuda:0")
    state = piso.make_state(dom, u0=g["u0"], device=dev)
    for b, ref in zip(state.bc, G.split_bc(g, g["bc0"])):
        b.copy_(torch.as_tensor(ref, device=dev))
    cfg = piso.StepConfig(dt=float(g["dt"]), nu=float(g["nu"]),
                          n_correctors=int(g["n_correctors"]),
                          nonortho_correctors=int(g["nonortho"]),
                          source=G.source_of(g), tol=tol)
    ws = piso.PisoWorkspace(dom)
    tapes, outs = [], []
    for _ in range(int(g["steps"])):
        tape = piso.StepTape()
        state, diag = piso.piso_step(dom, state, cfg, ws, tape)
        tapes.append(tape)
        outs.append((state, diag))
    return g, dom, tapes, outs


@pytest.mark.parametrize("name", G.ALL)
def test_forward_matches_reference(name):
    g, dom, tapes, outs = _gpu_rollout(name)
    for k, (st, diag) in enumerate(outs):
        assert G.rel(_np(st.u), g[f"s{k}_u"]) < FIELD_TOL
        assert G.rel(_np(st.p), g[f"s{k}_p"]) < FIELD_TOL
        assert G.rel(_np(tapes[k].c_data), g[f"s{k}_C"]) < FIELD_TOL
        assert G.rel(-_np(tapes[k].k_data), g[f"s{k}_P"]) < FIELD_TOL
        assert G.rel(_np(tapes[k].rhs_final), g[f"s{k}_rhs"]) < FIELD_TOL
        assert G.rel(_np(tapes[k].mom_iters[-1]), g[f"s{k}_ustar"]) \
            < FIELD_TOL
        for m, corr in enumerate(tapes[k].correctors):
            assert G.rel(_np(corr.h), g[f"s{k}_h{m}"]) < FIELD_TOL
            assert G.rel(_np(corr.p_iters[-1]), g[f"s{k}_p{m}"]) < FIELD_TOL
        if st.bc:
            bc = np.concatenate([_np(b) for b in st.bc])
            assert G.rel(bc, g[f"s{k}_bc"]) < FIELD_TOL
        assert diag.advout_scale == pytest.approx(
            float(g[f"s{k}_advout_scale"]), rel=1e-9, abs=1e-12)
        assert diag.div_wide_max == pytest.approx(
            float(g[f"s{k}_div_wide_max"]), rel=1e-6, abs=1e-9)
        assert diag.momentum_iterations > 0
        assert diag.pressure_iterations > 0


@pytest.mark.parametrize("name", G.ALL)
@pytest.mark.parametrize("path", ["full", "adv_only", "p_only", "none"])
def test_backward_matches_reference(name, path):
    from paper_2505_16992_b200 import adjoint
    g, dom, tapes, outs = _gpu_rollout(name)
    dev = torch.device("cuda:0")
    cot = adjoint.GradState(u=torch.as_tensor(g["cot_u"], device=dev),
                            p=torch.as_tensor(g["cot_p"], device=dev))
    cots = [None] * (len(tapes) - 1) + [cot]
    r = adjoint.backward_rollout(dom, tapes, cots, path=path, tol=GPU_TOL)
    key = f"g_{path}"
    assert G.rel(_np(r.u), g[key + "_u"]) < FIELD_TOL
    assert r.nu == pytest.approx(float(g[key + "_nu"]), rel=FIELD_TOL,
                                 abs=1e-12)
    assert G.rel(_np(r.source), g[key + "_source"]) < FIELD_TOL
    if r.bc:
        bc = np.concatenate([_np(b) for b in r.bc])
        assert G.rel(bc, g[key + "_bc"]) < FIELD_TOL
    if path == "none":
        assert r.solve_iterations == 0
    else:
        assert r.solve_iterations > 0


def test_backward_step_single_matches_reference():
    from paper_2505_16992_b200 import adjoint
    g, dom, tapes, outs = _gpu_rollout("channel")
    dev = torch.device("cuda:0")
    cot = adjoint.GradState(u=torch.as_tensor(g["cot_u"], device=dev),
                            p=torch.as_tensor(g["cot_p"], device=dev))
    r = adjoint.backward_step(dom, tapes[0], cot, tol=GPU_TOL)
    assert G.rel(_np(r.u), g["g1_u"]) < FIELD_TOL
    assert r.nu == pytest.approx(float(g["g1_nu"]), rel=FIELD_TOL)
    assert G.rel(_np(r.source), g["g1_source"]) < FIELD_TOL
    assert G.rel(np.concatenate([_np(b) for b in r.bc]), g["g1_bc"]) \
        < FIELD_TOL


def test_backward_bitwise_deterministic():
    from paper_2505_16992_b200 import adjoint
    g, dom, tapes, outs = _gpu_rollout("box3d")
    dev = torch.device("cuda:0")
    cot = adjoint.GradState(u=torch.as_tensor(g["cot_u"], device=dev),
                            p=torch.zeros(dom.n, dtype=torch.float64,
                                          device=dev))
    g1 = adjoint.backward_step(dom, tapes[-1], cot, tol=GPU_TOL)
    g2 = adjoint.backward_step(dom, tapes[-1], cot, tol=GPU_TOL)
    assert torch.equal(g1.u, g2.u)
    assert g1.nu == g2.nu
    assert torch.equal(g1.source, g2.source)


def test_zero_cotangent_gives_zero_gradient():
    from paper_2505_16992_b200 import adjoint
    g, dom, tapes, outs = _gpu_rollout("cavity8")
    for p in adjoint.GradientPath:
        r = adjoint.backward_step(dom, tapes[0],
                                  adjoint.GradState.zeros(dom), path=p)
        assert float(r.u.abs().max()) == 0.0
        assert r.nu == 0.0
        assert all(float(b.abs().max()) == 0.0 for b in r.bc)


@pytest.mark.parametrize("name", ["channel", "twoblock_rot", "obstacle"])
def test_stencil_matvec_and_transpose(name):
    from paper_2505_16992_b200 import linalg
    g = G.load(name)
    dom = G.build(name)
    plan = dom.device_plan("cuda:0")
    rng = np.random.default_rng(3)
    st = g["s0_C"]
    x = rng.standard_normal(dom.n)
    for tr in (False, True):
        y = linalg.stencil_matvec(plan, torch.as_tensor(st, device="cuda:0"),
                                  torch.as_tensor(x, device="cuda:0"),
                                  transpose=tr)
        ref = O.stencil_matvec(dom, st, x, transpose=tr)
        assert G.rel(_np(y), ref) < 1e-14


@pytest.mark.parametrize("name", ["channel", "refined_cavity", "obstacle"])
def test_cg_matches_oracle_krylov_iterations(name):
    """Same Jacobi-PCG recurrence as the oracle restatement: same solution
    and the same iteration count (+-1 for round-off at the threshold)."""
    from paper_2505_16992_b200 import linalg
    g = G.load(name)
    dom = G.build(name)
    plan = dom.device_plan("cuda:0")
    K = -g["s0_P"]
    rng = np.random.default_rng(5)
    b = rng.standard_normal(dom.n)
    x_o, ok_o, it_o = O.cg(dom, K, b, tol=1e-10)
    x, rep = linalg.cg_solve(plan, torch.as_tensor(K, device="cuda:0"),
                             torch.as_tensor(b, device="cuda:0"), tol=1e-10,
                             zero_mean=True, precond="jacobi")
    assert rep.converged and ok_o
    assert abs(rep.iterations - it_o) <= 1
    assert G.rel(_np(x), x_o) < 1e-8


def _pressure_operator(dom, seed=4):
    """K = -P of the oracle for a random velocity (host, exact restatement)."""
    rng = np.random.default_rng(seed)
    u = 0.3 * rng.standard_normal((dom.n, dom.dim))
    C = O.assemble_momentum(dom, u, 0.01, 0.05)
    return -O.assemble_pressure(dom, 1.0 / C[0])


MG_DOMAINS = {
    "channel8": lambda: __import__("paper_2505_16992_b200.mesh", fromlist=["m"])
    .make_channel((8, 8, 4), ratio=1.1),
    "channel16": lambda: __import__("paper_2505_16992_b200.mesh",
                                    fromlist=["m"])
    .make_channel((16, 12, 8), ratio=1.03),
    "refined_cavity": lambda: G.build("refined_cavity"),
    "cavity8": lambda: G.build("cavity8"),
    "sheared3d": lambda: G.build("sheared3d"),
}


def _plan(dom, geom):
    from paper_2505_16992_b200.plan import DevicePlan
    return DevicePlan(dom, torch.device("cuda", 0), geom_precond=geom)


@pytest.mark.parametrize("name", sorted(MG_DOMAINS))
def test_multigrid_pcg_converges_to_exact_solution(name):
    """The multigrid-preconditioned CG (the GPU's ILU(0) replacement) lands
    on the same zero-mean solution as the exact oracle, needs fewer
    iterations than Jacobi, and is bitwise reproducible (block-Jacobi line
    smoothing and fixed-order reductions)."""
    from paper_2505_16992_b200 import linalg
    dom = MG_DOMAINS[name]()
    plan = _plan(dom, "multigrid")
    assert plan.has_mg and plan.mg_levels >= 2
    assert plan.geom_kind == "multigrid"
    K = _pressure_operator(dom)
    rng = np.random.default_rng(7)
    b = rng.standard_normal(dom.n)
    Kt = torch.as_tensor(K, device="cuda:0")
    bt = torch.as_tensor(b, device="cuda:0")
    x, rep = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                             precond="mg")
    xj, repj = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                               precond="jacobi")
    x_exact = O.solve_pressure_exact(dom, K, b)
    assert rep.converged and not rep.fallback_used
    assert G.rel(_np(x), x_exact) < 1e-8
    assert abs(float(x.mean())) < 1e-12
    assert rep.iterations < repj.iterations
    x2, rep2 = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                               precond="mg")
    assert torch.equal(x, x2) and rep2.iterations == rep.iterations


@pytest.mark.parametrize("shape", [(32, 32), (64, 48)])
def test_multigrid_staged_coarse_cycle_matches_global(shape, monkeypatch):
    """Small hierarchies run their coarse V-cycle from shared memory
    (k_mg_coarse_staged); PF_MG_NO_STAGE=1 runs the same cycle on global
    memory (k_mg_coarse_fused).  Same arithmetic per line and cell, so the
    solves agree to rounding (the coarsest mean is reduced over a different
    block size) with the same iteration counts, and both land on the exact
    solution."""
    from paper_2505_16992_b200 import linalg, mesh
    dom = mesh.make_cavity(shape)
    plan = _plan(dom, "multigrid")
    assert plan.has_mg and plan.mg_levels >= 3
    K = _pressure_operator(dom)
    b = np.random.default_rng(3).standard_normal(dom.n)
    Kt = torch.as_tensor(K, device="cuda:0")
    bt = torch.as_tensor(b, device="cuda:0")
    x_exact = O.solve_pressure_exact(dom, K, b)
    out = {}
    for staged in (True, False):
        if staged:
            monkeypatch.delenv("PF_MG_NO_STAGE", raising=False)
        else:
            monkeypatch.setenv("PF_MG_NO_STAGE", "1")
        x, rep = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                                 precond="mg")
        assert rep.converged and not rep.fallback_used
        assert G.rel(_np(x), x_exact) < 1e-8
        out[staged] = (_np(x), rep.iterations)
    assert abs(out[True][1] - out[False][1]) <= 1
    assert G.rel(out[True][0], out[False][0]) < 1e-9


SPECTRAL_DOMAINS = {
    "channel8": MG_DOMAINS["channel8"],
    "channel16": MG_DOMAINS["channel16"],
    "channel_long": lambda: __import__("paper_2505_16992_b200.mesh",
                                       fromlist=["m"])
    .make_channel((32, 10, 4), ratio=1.2),
    "channel_wide": lambda: __import__("paper_2505_16992_b200.mesh",
                                       fromlist=["m"])
    .make_channel((4, 16, 64), ratio=1.05),
    # length-256 X / Z: the register four-step FFT kernels
    "channel_z256": lambda: __import__("paper_2505_16992_b200.mesh",
                                       fromlist=["m"])
    .make_channel((4, 8, 256), ratio=1.1),
    "channel_x256": lambda: __import__("paper_2505_16992_b200.mesh",
                                       fromlist=["m"])
    .make_channel((256, 6, 8), ratio=1.1),
}


@pytest.mark.parametrize("name", sorted(SPECTRAL_DOMAINS))
def test_spectral_pcg_converges_to_exact_solution(name):
    """The spectral preconditioner (FFT in the periodic X / Z, tridiagonal
    in Y) lands on the exact zero-mean solution, deterministically, and
    beats Jacobi even on an operator far from plane-uniform."""
    from paper_2505_16992_b200 import linalg
    dom = SPECTRAL_DOMAINS[name]()
    plan = _plan(dom, "auto")
    assert plan.has_mg and plan.geom_kind == "spectral"
    K = _pressure_operator(dom)
    b = np.random.default_rng(7).standard_normal(dom.n)
    Kt = torch.as_tensor(K, device="cuda:0")
    bt = torch.as_tensor(b, device="cuda:0")
    x, rep = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                             precond="mg")
    xj, repj = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                               precond="jacobi")
    x_exact = O.solve_pressure_exact(dom, K, b)
    assert rep.converged and not rep.fallback_used
    assert G.rel(_np(x), x_exact) < 1e-8
    assert abs(float(x.mean())) < 1e-12
    assert rep.iterations < repj.iterations
    x2, rep2 = linalg.cg_solve(plan, Kt, bt, tol=1e-11, zero_mean=True,
                               precond="mg")
    assert torch.equal(x, x2) and rep2.iterations == rep.iterations


@pytest.mark.parametrize("name", sorted(SPECTRAL_DOMAINS))
def test_spectral_is_exact_inverse_of_plane_uniform_operator(name):
    """With u = 0 the momentum diagonal depends on Y only, so K is exactly
    diagonalised by the transforms: the spectral-PCG needs at most 2
    iterations to 1e-11 (one, up to round-off)."""
    from paper_2505_16992_b200 import linalg
    dom = SPECTRAL_DOMAINS[name]()
    plan = _plan(dom, "auto")
    C = O.assemble_momentum(dom, np.zeros((dom.n, dom.dim)), 0.01, 0.05)
    K = -O.assemble_pressure(dom, 1.0 / C[0])
    b = np.random.default_rng(11).standard_normal(dom.n)
    x, rep = linalg.cg_solve(plan, torch.as_tensor(K, device="cuda:0"),
                             torch.as_tensor(b, device="cuda:0"), tol=1e-11,
                             zero_mean=True, precond="mg")
    assert rep.converged and rep.iterations <= 2
    assert G.rel(_np(x), O.solve_pressure_exact(dom, K, b)) < 1e-9


def test_spectral_falls_back_to_multigrid():
    """Non-power-of-two periodic X (6): the plan picks multigrid."""
    plan = _plan(G.build("channel"), "auto")
    assert plan.geom_kind == "multigrid"


def test_multigrid_odd_periodic_coarsest_with_jacobi_lines():
    """(6, 8, 4) coarsens x to 3 (odd, periodic): fine for the default
    block-Jacobi smoother (the red-black one refuses such grids)."""
    from paper_2505_16992_b200 import linalg
    dom = G.build("channel")
    plan = dom.device_plan("cuda:0")
    assert plan.has_mg
    K = _pressure_operator(dom)
    b = np.random.default_rng(9).standard_normal(dom.n)
    x, rep = linalg.cg_solve(plan, torch.as_tensor(K, device="cuda:0"),
                             torch.as_tensor(b, device="cuda:0"), tol=1e-11,
                             zero_mean=True, precond="mg")
    assert rep.converged
    assert G.rel(_np(x), O.solve_pressure_exact(dom, K, b)) < 1e-8


def test_multigrid_hierarchy_reused_and_rebuilt():
    from paper_2505_16992_b200 import linalg, mesh
    dom = mesh.make_channel((8, 8, 4), ratio=1.1)
    plan = dom.device_plan("cuda:0")
    K = torch.as_tensor(_pressure_operator(dom), device="cuda:0")
    b = torch.as_tensor(np.random.default_rng(8).standard_normal(dom.n),
                        device="cuda:0")
    x1, _ = linalg.cg_solve(plan, K, b, tol=1e-12, zero_mean=True)
    key = plan._mg_key
    x2, _ = linalg.cg_solve(plan, K, b, tol=1e-12, zero_mean=True)
    assert plan._mg_key == key
    assert torch.equal(x1, x2)
    K2 = K.clone()
    K2.mul_(2.0)                      # same values scaled: a new operator
    x3, _ = linalg.cg_solve(plan, K2, b, tol=1e-12, zero_mean=True)
    assert plan._mg_key != key
    assert G.rel(_np(x3), _np(x1) / 2.0) < 1e-9


@pytest.mark.parametrize("name", ["channel", "backstep"])
def test_bicgstab_matches_oracle_krylov(name):
    from paper_2505_16992_b200 import linalg
    g = G.load(name)
    dom = G.build(name)
    plan = dom.device_plan("cuda:0")
    C = g["s0_C"]
    rng = np.random.default_rng(6)
    b = rng.standard_normal((dom.dim, dom.n))
    x, reps = linalg.bicgstab_solve(plan, torch.as_tensor(C, device="cuda:0"),
                                    torch.as_tensor(b, device="cuda:0"),
                                    tol=1e-12, precond="jacobi")
    for c in range(dom.dim):
        xo, ok, it = O.bicgstab(dom, C, b[c], tol=1e-12)
        assert reps[c].converged and ok
        assert abs(reps[c].iterations - it) <= 1
        assert G.rel(_np(x[c]), xo) < 1e-9
    # transposed system
    xt, reps = linalg.bicgstab_solve(plan, torch.as_tensor(C, device="cuda:0"),
                                     torch.as_tensor(b, device="cuda:0"),
                                     tol=1e-12, transpose=True)
    for c in range(dom.dim):
        xo = O.solve_exact(dom, C, b[c], transpose=True)
        assert G.rel(_np(xt[c]), xo) < 1e-9


def test_solver_error_on_nonconvergence():
    from paper_2505_16992_b200 import linalg
    g = G.load("channel")
    dom = G.build("channel")
    plan = dom.device_plan("cuda:0")
    K = torch.as_tensor(-g["s0_P"], device="cuda:0")
    b = torch.as_tensor(np.random.default_rng(0).standard_normal(dom.n),
                        device="cuda:0")
    with pytest.raises(linalg.SolverError) as ei:
        linalg.cg_solve(plan, K, b, tol=1e-14, maxiter=2, zero_mean=True,
                        stage="pressure[c0i0]")
    rep = ei.value.report
    assert not rep.converged and rep.fallback_used
    assert rep.stage == "pressure[c0i0]"
    assert rep.iterations == 2 + 4


def test_zero_rhs_returns_zero():
    from paper_2505_16992_b200 import linalg
    dom = G.build("cavity8")
    plan = dom.device_plan("cuda:0")
    K = torch.as_tensor(-G.load("cavity8")["s0_P"], device="cuda:0")
    x, rep = linalg.cg_solve(plan, K, torch.zeros(dom.n, dtype=torch.float64,
                                                  device="cuda:0"),
                             x0=torch.ones(dom.n, dtype=torch.float64,
                                           device="cuda:0"), zero_mean=True)
    assert rep.converged and rep.iterations == 0 and rep.residual == 0.0
    assert float(x.abs().max()) == 0.0


def test_nonorthogonal_plan_carries_cross_terms():
    dom = G.build("distorted_nonortho")
    plan = dom.device_plan("cuda:0")
    assert plan.nonortho and plan.cell_cross
    assert plan.alpha_full is not None and plan.finfo is not None


def test_step_validates_dt_nu():
    from paper_2505_16992_b200 import piso
    dom = G.build("cavity8")
    st = piso.make_state(dom, device="cuda:0")
    with pytest.raises(ValueError):
        piso.piso_step(dom, st, piso.StepConfig(dt=0.0, nu=0.1))
    with pytest.raises(ValueError):
        piso.piso_step(dom, st, piso.StepConfig(dt=0.1, nu=-1.0))


def test_shear_mode_exact_implicit_decay():
    """Known answer (T/test_piso.py:56-73): one step damps the periodic
    shear mode by exactly 1/(1 + nu k^2 dt)."""
    from paper_2505_16992_b200 import mesh, piso
    nx, ny = 6, 16
    dom = mesh.make_box((nx, ny))
    y = dom.centers[:, 1]
    eps, nu, dt = 1e-3, 0.3, 0.7
    u0 = np.zeros((dom.n, 2))
    u0[:, 0] = eps * np.sin(2 * np.pi * y / ny)
    st = piso.make_state(dom, u0=u0, device="cuda:0")
    new, diag = piso.piso_step(dom, st, piso.StepConfig(dt=dt, nu=nu,
                                                        tol=1e-12))
    k2 = 2.0 - 2.0 * np.cos(2 * np.pi / ny)
    expected = u0[:, 0] / (1.0 + nu * k2 * dt)
    assert np.allclose(_np(new.u[:, 0]), expected, atol=1e-12)
    assert float(new.u[:, 1].abs().max()) < 1e-12
    assert float(new.p.abs().max()) < 1e-10
