"""Child process of test_gpu_cg_single.py: the pressure CG variant is chosen
once per process (PF_CG_VARIANT), so each variant solves the same systems in
its own interpreter and writes solutions + reports to an .npz."""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import golden_cases as G  # noqa: E402
from oracle import pisoref as O  # noqa: E402


def pressure_operator(dom, seed=4):
    rng = np.random.default_rng(seed)
    u = 0.3 * rng.standard_normal((dom.n, dom.dim))
    C = O.assemble_momentum(dom, u, 0.01, 0.05)
    return -O.assemble_pressure(dom, 1.0 / C[0])


def domains():
    from paper_2505_16992_b200 import mesh
    return {
        # multigrid preconditioner
        "cavity8": (lambda: G.build("cavity8"), "multigrid"),
        "sheared3d": (lambda: G.build("sheared3d"), "multigrid"),
        "channel16_mg": (lambda: mesh.make_channel((16, 12, 8), ratio=1.03),
                         "multigrid"),
        # spectral preconditioner; (32, 16, 32) has whole 8 x 32 Y/Z tiles
        # (the classic variant runs the tiled CG there)
        "channel16": (lambda: mesh.make_channel((16, 12, 8), ratio=1.03),
                      "auto"),
        "channel_tiled": (lambda: mesh.make_channel((32, 16, 32), ratio=1.1),
                          "auto"),
    }


def main(out):
    from paper_2505_16992_b200 import linalg
    from paper_2505_16992_b200.plan import DevicePlan
    res = {}
    for name, (build, geom) in domains().items():
        dom = build()
        plan = DevicePlan(dom, torch.device("cuda", 0), geom_precond=geom)
        K = torch.as_tensor(pressure_operator(dom), device="cuda:0")
        b = torch.as_tensor(np.random.default_rng(7).standard_normal(dom.n),
                            device="cuda:0")
        for tol in (1e-8, 1e-11):
            x, rep = linalg.cg_solve(plan, K, b, tol=tol, zero_mean=True,
                                     precond="mg")
            # warm start from the solution of a perturbed right-hand side
            x2, rep2 = linalg.cg_solve(plan, K, 1.01 * b, x0=x, tol=tol,
                                       zero_mean=True, precond="mg")
            key = f"{name}_{tol:g}"
            res[key + "_x"] = x.cpu().numpy()
            res[key + "_x2"] = x2.cpu().numpy()
            res[key + "_rep"] = np.array(
                [rep.iterations, rep.converged, rep.residual,
                 rep2.iterations, rep2.converged, rep2.residual],
                dtype=np.float64)
        # a zero right-hand side and maxiter 0 / 1 edge cases
        z, repz = linalg.cg_solve(plan, K, torch.zeros_like(b), tol=1e-8,
                                  zero_mean=True, precond="mg")
        res[name + "_zero"] = np.array([repz.iterations, repz.converged,
                                        float(z.abs().max())])
        x1, rep1 = linalg.cg_solve(plan, K, b, tol=1e-12, maxiter=1,
                                   zero_mean=True, precond="mg",
                                   raise_on_fail=False)
        res[name + "_max1"] = np.array([rep1.iterations, rep1.converged])
        res[name + "_max1_x"] = x1.cpu().numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
