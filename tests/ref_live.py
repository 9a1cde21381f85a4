"""Run the reference itself (``pisoflow``, built unmodified into
``oracle/_ref`` by ``oracle/build_ref.py``) next to the CUDA path on the
same inputs.  TEST INFRASTRUCTURE: the reference is the checker, never the
thing measured.  ``oracle/_ref`` is git-ignored but travels to the GPU box
with the repository snapshot; ``/root/reference`` is never read here.

Each case builds the SAME workload through both APIs (the reference's
``pisoflow.mesh`` generators and this package's mirrors), feeds the
reference's initial state to both, runs K taped steps with warm starts
(the reference's ``run_rollout`` setting, S/cases.py:183) and a
``backward_rollout`` (S/adjoint.py:509-539) with per-step cotangents, and
returns both sides' fields, gradients and solver iteration counts.
"""

import os
import sys

import numpy as np


def reference():
    """Import the reference package from oracle/_ref (compiled lane)."""
    from oracle import build_ref
    build_ref.build()
    path = build_ref.ref_path()
    if not os.path.isdir(os.path.join(path, "pisoflow")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import pisoflow  # noqa: F401
    from pisoflow import adjoint, kernels, mesh, piso
    return {"adjoint": adjoint, "kernels": kernels, "mesh": mesh,
            "piso": piso}


def rel(a, b):
    """L-inf error relative to max|b| (SURVEY.md §8 c)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


# ---------------------------------------------------------------------------
# workloads (both sides build the same grid through their own generators)


def channel(M, shape=(64, 48, 64), ratio=1.03):
    """C4's recipe at a smaller size: make_channel + reichardt_init(Re_tau
    180, perturbation 0.1, seed 0) + per-step wall forcing; dt = 0.3 (2 pi /
    nx) / max|u0| (SURVEY.md §8 d)."""
    dom = M.make_channel(shape, ratio=ratio)
    return dom


def refined_cavity(M, n=128, ratio=1.03, lid_speed=1.0):
    """C2's grid at a smaller size: [0,1]^2 wall-refined on both axes, lid
    y = 1 moving +x (SURVEY.md §8 d)."""
    x = M.wall_refined_coords(n, 0.5, ratio)
    blk = M.BlockSpec(M._grid_vertices(x, x))
    bnd = {(0, a, s): M.Dirichlet(0.0) for a in range(2) for s in (0, 1)}
    bnd[(0, 1, 1)] = M.Dirichlet((lid_speed, 0.0))
    return M.Domain([blk], bnd), float(np.diff(x).min())


def obstacle(M, q=8):
    """C3's 8-block obstacle grid at q cells per unit (C3 uses 64): 32 x 8
    domain, 1 x 1 obstacle centred at (6.5, 4), uniform inflow."""
    def inlet(fc):
        return np.stack([np.ones(len(fc)), np.zeros(len(fc))], axis=-1)
    return M.make_obstacle_grid(domain_size=(32.0, 8.0),
                                obstacle_center=(6.5, 4.0),
                                obstacle_size=(1.0, 1.0),
                                nx=(6 * q, q, 25 * q), ny=(7 * q // 2, q,
                                                           7 * q // 2),
                                inlet=inlet)


def face_index(domain, axis, side):
    return next(i for i, f in enumerate(domain.bfaces)
                if f.axis == axis and f.side == side)
