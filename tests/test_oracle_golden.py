"""CPU tier: pin the oracle and this repository's Domain against golden
vectors produced by the reference implementation itself."""

import numpy as np
import pytest

import golden_cases as G
from oracle import pisoref as O

TOL = 1e-10   # golden vectors were produced at solver tol 1e-13


@pytest.mark.parametrize("name", G.ALL)
def test_domain_matches_reference_mesh(name):
    g = G.load(name)
    dom = G.build(name)
    assert dom.n == g["jac"].shape[0]
    np.testing.assert_array_equal(dom.nbr, g["nbr"])
    np.testing.assert_array_equal(dom.nbr_ax, g["nbr_ax"])
    np.testing.assert_array_equal(dom.nbr_sign, g["nbr_sign"])
    assert G.rel(dom.jac, g["jac"]) < 1e-14
    assert G.rel(dom.tmat, g["tmat"]) < 1e-14
    assert G.rel(dom.alpha, g["alpha"]) < 1e-14
    assert G.rel(dom.centers, g["centers"]) < 1e-15
    np.testing.assert_array_equal([f.m for f in dom.bfaces], g["bface_m"])
    if dom.bfaces:
        assert G.rel(np.concatenate([f.face_jac for f in dom.bfaces]),
                     g["bface_jac"]) < 1e-14
        assert G.rel(np.concatenate([f.face_t for f in dom.bfaces]),
                     g["bface_t"]) < 1e-14
        assert G.rel(np.concatenate([f.face_alpha for f in dom.bfaces]),
                     g["bface_alpha"]) < 1e-14


def test_nonorthogonal_detection():
    assert G.build("distorted_nonortho").has_cross_terms()
    for name in G.ORTHOGONAL:
        assert not G.build(name).has_cross_terms(), name


def _oracle_rollout(name):
    g = G.load(name)
    dom = G.build(name)
    bc0 = G.split_bc(g, g["bc0"])
    tapes, outs = O.rollout(dom, g["u0"], bc0, float(g["dt"]),
                            float(g["nu"]), int(g["steps"]),
                            source=G.source_of(g),
                            n_correctors=int(g["n_correctors"]))
    return g, dom, tapes, outs


@pytest.mark.parametrize("name", G.ORTHOGONAL)
def test_oracle_forward_matches_reference(name):
    g, dom, tapes, outs = _oracle_rollout(name)
    for k, (u, p, bc, dg) in enumerate(outs):
        assert G.rel(u, g[f"s{k}_u"]) < TOL
        assert G.rel(p, g[f"s{k}_p"]) < 1e-9
        # step 0 matrices depend on inputs only; later ones on solved fields
        mt = 1e-13 if k == 0 else TOL
        assert G.rel(tapes[k].C, g[f"s{k}_C"]) < mt
        assert G.rel(-tapes[k].K, g[f"s{k}_P"]) < mt
        assert G.rel(tapes[k].rhs, g[f"s{k}_rhs"]) < mt
        assert G.rel(tapes[k].u_star, g[f"s{k}_ustar"]) < TOL
        for m, (_, h, pm) in enumerate(tapes[k].correctors):
            assert G.rel(h, g[f"s{k}_h{m}"]) < TOL
        if len(bc):
            assert G.rel(np.concatenate(bc), g[f"s{k}_bc"]) < 1e-12
        assert abs(dg["advout_scale"] - float(g[f"s{k}_advout_scale"])) \
            < 1e-12
        assert abs(dg["div_wide_max"] - float(g[f"s{k}_div_wide_max"])) \
            <= 1e-8 * max(1.0, float(g[f"s{k}_div_wide_max"]))


@pytest.mark.parametrize("name", G.ORTHOGONAL)
@pytest.mark.parametrize("path", ["full", "adv_only", "p_only", "none"])
def test_oracle_backward_matches_reference(name, path):
    g, dom, tapes, outs = _oracle_rollout(name)
    r = O.backward_rollout(dom, tapes, g["cot_u"], g["cot_p"], path)
    key = f"g_{path}"
    assert G.rel(r["u"], g[key + "_u"]) < TOL
    assert abs(r["nu"] - float(g[key + "_nu"])) <= TOL * max(
        1.0, abs(float(g[key + "_nu"])))
    assert G.rel(r["source"], g[key + "_source"]) < TOL
    if r["bc"]:
        assert G.rel(np.concatenate(r["bc"]), g[key + "_bc"]) < TOL


def test_oracle_krylov_restatement_converges_to_exact():
    g, dom, tapes, outs = _oracle_rollout("channel")
    t = tapes[0]
    b = -O.divergence_rhs(dom, t.correctors[0][1], t.bc)
    x_exact = O.solve_pressure_exact(dom, t.K, b)
    x, ok, it = O.cg(dom, t.K, b, tol=1e-12)
    assert ok and it > 0
    assert G.rel(x, x_exact) < 1e-9
    y, ok, it = O.bicgstab(dom, t.C, t.rhs[:, 0], tol=1e-12)
    assert ok
    assert G.rel(y, t.u_star[:, 0]) < 1e-10


@pytest.mark.parametrize("case", ["channel", "cavity8", "obstacle"])
def test_oracle_single_reduction_cg_matches_classic(case):
    """The product's single-reduction (Chronopoulos-Gear) pressure CG, the
    slab plans' variant, restated in the oracle: the same iterates as the
    reference's loop (S/linalg.py:136-170) up to rounding -- same iteration
    count within one, same solution to the solve's accuracy."""
    g, dom, tapes, outs = _oracle_rollout(case)
    t = tapes[0]
    b = -O.divergence_rhs(dom, t.correctors[0][1], t.bc)
    for pc in ("jacobi", None):
        xc, okc, itc = O.cg(dom, t.K, b, tol=1e-10, precond=pc)
        xs, oks, its = O.cg(dom, t.K, b, tol=1e-10, precond=pc,
                            variant="single")
        assert okc and oks and abs(itc - its) <= 1, (pc, itc, its)
        assert G.rel(xs, xc) < 1e-7, (pc, G.rel(xs, xc))
        assert abs(xs.mean()) < 1e-12 * max(1.0, np.abs(xs).max())


@pytest.mark.parametrize("transpose", [False, True])
def test_oracle_neumann2_restatement(transpose):
    """The two-sweep Jacobi polynomial preconditioner of the product's
    BiCGStab (csrc/bicg_nm.cuh) in the oracle's Krylov restatement: same
    solution as the exact solve, fewer iterations than Jacobi."""
    g = G.load("channel")
    dom = G.build("channel")
    C = g["s0_C"]
    b = np.random.default_rng(0).standard_normal(dom.n)
    ex = O.solve_exact(dom, C, b, transpose=transpose)
    xj, okj, itj = O.bicgstab(dom, C, b, tol=1e-12, transpose=transpose)
    xn, okn, itn = O.bicgstab(dom, C, b, tol=1e-12, precond="neumann2",
                              transpose=transpose)
    assert okj and okn and itn < itj
    assert G.rel(xn, ex) < 1e-10
