"""Generate golden vectors from the REFERENCE implementation (test fixture).

Run in the build container, where ``/root/reference`` exists:

    python oracle/build_ref.py            # compiled reference lane -> oracle/_ref
    python tests/golden/make_golden.py    # writes tests/golden/*.npz

Each case builds a mesh with the reference's own generators, runs a short
taped rollout with ``pisoflow.piso.piso_step`` at a tight solver tolerance
and reverses it with ``pisoflow.adjoint.backward_rollout``; the arrays are
stored with the momentum / pressure matrices converted from the reference's
CSR ``data`` to the (2d+1, n) stencil layout used by this repository
(row 0 diagonal, row 1 + 2a + s the neighbour across face (a, s)).

The fixtures are the parity anchor that travels to the GPU box (the
reference itself does not); the committed .npz files were produced by this
script and are loaded by tests/test_oracle_golden.py and the GPU parity
tests.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import build_ref  # noqa: E402

build_ref.build()
sys.path.insert(0, build_ref.ref_path())

from pisoflow import adjoint, mesh, piso  # noqa: E402
from pisoflow.kernels import LANE  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from golden_cases import sheared3d  # noqa: E402

TOL = 1e-13


def stencil(dom, data):
    d, n = dom.dim, dom.n
    out = np.zeros((2 * d + 1, n))
    out[0] = data[dom.pattern.diag_pos]
    for a in range(d):
        for s in (0, 1):
            ok = dom.nb_slot[a, s] >= 0
            out[1 + 2 * a + s, ok] = data[dom.nb_slot[a, s, ok]]
    return out


def cases():
    rng = np.random.default_rng(20251017)

    def rand(shape, scale):
        return scale * rng.standard_normal(shape)

    out = []
    dom = mesh.make_cavity((8, 8))
    out.append(("cavity8", dom, dict(dt=0.05, nu=0.05),
                rand((dom.n, 2), 0.2), None, 3))
    dom = mesh.make_box((4, 5, 6))
    out.append(("box3d", dom, dict(dt=0.1, nu=0.2, source=(0.3, -0.1, 0.2)),
                rand((dom.n, 3), 0.3), None, 2))
    dom = mesh.make_channel((6, 8, 4), ratio=1.1)
    out.append(("channel", dom, dict(dt=0.05, nu=0.01),
                rand((dom.n, 3), 0.5), rand((dom.n, 3), 0.1), 2))
    dom = mesh.make_two_block((4, 4), rotated=True)
    out.append(("twoblock_rot", dom, dict(dt=0.07, nu=0.2,
                                          source=(1.0, 0.2)),
                rand((dom.n, 2), 0.2), None, 2))
    dom = mesh.make_backstep(cells_per_h=2)
    out.append(("backstep", dom, dict(dt=0.05, nu=0.05),
                rand((dom.n, 2), 0.1), None, 2))
    dom = mesh.make_obstacle_grid(nx=(4, 3, 8), ny=(4, 3, 4))
    out.append(("obstacle", dom, dict(dt=0.05, nu=0.05),
                rand((dom.n, 2), 0.1), None, 2))
    coords = mesh.wall_refined_coords(12, 0.5, 1.2)
    blk = mesh.BlockSpec(mesh._grid_vertices(coords, coords))
    bnd = {(0, a, s): mesh.Dirichlet(0.0) for a in range(2) for s in (0, 1)}
    bnd[(0, 1, 1)] = mesh.Dirichlet((1.0, 0.0))
    dom = mesh.Domain([blk], bnd)
    out.append(("refined_cavity", dom, dict(dt=0.01, nu=0.01),
                rand((dom.n, 2), 0.1), None, 2))
    dom = mesh.make_poiseuille((6, 4), distort=0.35)
    out.append(("distorted_nonortho", dom,
                dict(dt=0.07, nu=0.2, nonortho_correctors=1),
                rand((dom.n, 2), 0.3), None, 2))
    dom = sheared3d(mesh)
    out.append(("sheared3d", dom,
                dict(dt=0.05, nu=0.1, nonortho_correctors=2),
                rand((dom.n, 3), 0.2), rand((dom.n, 3), 0.1), 2))
    return out, rng


def run_case(name, dom, cfgkw, u0, src, steps, rng):
    d, n = dom.dim, dom.n
    cfg = piso.StepConfig(tol=TOL, source=src if src is not None
                          else cfgkw.pop("source", None), **cfgkw)
    state = piso.make_state(dom, u0=u0)
    ws = piso.PisoWorkspace(dom)
    rec = {"name": np.array(name), "lane": np.array(LANE),
           "steps": np.array(steps), "u0": u0,
           "dt": np.array(cfg.dt), "nu": np.array(cfg.nu),
           "n_correctors": np.array(cfg.n_correctors),
           "nonortho": np.array(cfg.nonortho_correctors),
           "tol": np.array(TOL)}
    src_arr = piso._resolve_source(dom, cfg.source)
    rec["source"] = src_arr
    rec["source_given"] = (np.asarray(cfg.source) if cfg.source is not None
                           else np.zeros(0))
    # mesh data for Domain parity
    rec["jac"], rec["tmat"], rec["alpha"] = dom.jac, dom.tmat, dom.alpha
    rec["centers"] = dom.centers
    rec["nbr"], rec["nbr_ax"], rec["nbr_sign"] = (dom.nbr, dom.nbr_ax,
                                                  dom.nbr_sign)
    rec["bc0"] = np.concatenate(state.bc, axis=0) if state.bc else \
        np.zeros((0, d))
    rec["bface_m"] = np.array([f.m for f in dom.bfaces])
    if dom.bfaces:
        rec["bface_jac"] = np.concatenate([f.face_jac for f in dom.bfaces])
        rec["bface_t"] = np.concatenate([f.face_t for f in dom.bfaces])
        rec["bface_alpha"] = np.concatenate([f.face_alpha
                                             for f in dom.bfaces])
    else:
        rec["bface_jac"] = np.zeros(0)
        rec["bface_t"] = np.zeros((0, d, d))
        rec["bface_alpha"] = np.zeros((0, d, d))
    tapes = []
    for k in range(steps):
        tape = piso.StepTape()
        state, dg = piso.piso_step(dom, state, cfg, ws, tape)
        tapes.append(tape)
        rec[f"s{k}_u"] = state.u
        rec[f"s{k}_p"] = state.p
        rec[f"s{k}_bc"] = (np.concatenate(state.bc, axis=0) if state.bc
                           else np.zeros((0, d)))
        rec[f"s{k}_C"] = stencil(dom, tape.c_data)
        rec[f"s{k}_P"] = stencil(dom, tape.p_data)
        rec[f"s{k}_rhs"] = tape.rhs_final
        rec[f"s{k}_ustar"] = tape.mom_iters[-1]
        for m, corr in enumerate(tape.correctors):
            rec[f"s{k}_h{m}"] = corr.h
            rec[f"s{k}_p{m}"] = corr.p_iters[-1]
        rec[f"s{k}_div_wide_max"] = np.array(dg.div_wide_max)
        rec[f"s{k}_advout_scale"] = np.array(dg.advout_scale)
        rec[f"s{k}_mom_iters"] = np.array(dg.momentum_iterations)
        rec[f"s{k}_p_iters"] = np.array(dg.pressure_iterations)
    wu = rng.standard_normal((n, d))
    wp = rng.standard_normal(n)
    rec["cot_u"], rec["cot_p"] = wu, wp
    for path in adjoint.GradientPath:
        cots = [None] * (steps - 1) + [adjoint.GradState(u=wu, p=wp)]
        g = adjoint.backward_rollout(dom, tapes, cots, path=path, tol=TOL)
        key = f"g_{path.value}"
        rec[key + "_u"] = g.u
        rec[key + "_nu"] = np.array(g.nu)
        rec[key + "_source"] = g.source
        rec[key + "_bc"] = (np.concatenate(g.bc, axis=0) if g.bc
                            else np.zeros((0, d)))
        rec[key + "_iters"] = np.array(g.solve_iterations)
    # single-step backward of the first step (stage-level anchor)
    g1 = adjoint.backward_step(dom, tapes[0], adjoint.GradState(u=wu, p=wp),
                               tol=TOL)
    rec["g1_u"], rec["g1_nu"] = g1.u, np.array(g1.nu)
    rec["g1_source"] = g1.source
    rec["g1_bc"] = (np.concatenate(g1.bc, axis=0) if g1.bc
                    else np.zeros((0, d)))
    return rec


def reichardt_fixture():
    """reichardt_init + wall_forcing_source on small channels."""
    rec = {}
    for tag, shape, ratio in (("a", (6, 8, 4), 1.1), ("b", (8, 12, 6), 1.03)):
        dom = mesh.make_channel(shape, ratio=ratio)
        st, nu, ut = piso.reichardt_init(dom, 180.0, perturbation=0.1,
                                         seed=3)
        rec[f"{tag}_u"], rec[f"{tag}_nu"] = st.u, np.array(nu)
        rec[f"{tag}_utau"] = np.array(ut)
        rec[f"{tag}_forcing"] = piso.wall_forcing_source(dom, st.u, nu)
        rec[f"{tag}_shape"], rec[f"{tag}_ratio"] = np.array(shape), \
            np.array(ratio)
    np.savez_compressed(os.path.join(HERE, "reichardt.npz"), **rec)
    print("reichardt fixture written")


def main():
    reichardt_fixture()
    all_cases, rng = cases()
    for name, dom, cfgkw, u0, src, steps in all_cases:
        rec = run_case(name, dom, dict(cfgkw), u0, src, steps, rng)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(f"{name}: n={dom.n} steps={steps} -> {os.path.getsize(path)} B")


if __name__ == "__main__":
    main()
