"""Prototype (CPU, scipy): BiCGStab iteration counts of the momentum solves
and their adjoints on a C4-spacing channel slab with Jacobi, wall-normal
line (Y-tridiagonal block-Jacobi) and the reference's ILU(0).  Systems are
captured from the reference's own piso_step / backward_step."""
import math
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, "/root/repo")
from oracle import build_ref  # noqa: E402
sys.path.insert(0, build_ref.ref_path())
from pisoflow import adjoint, linalg, mesh, piso  # noqa: E402

NX, NY, NZ = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3
                               else (32, 192, 32))]
x = np.arange(NX + 1) * (2 * np.pi / 256)
y = mesh.wall_refined_coords(NY, 1.0, 1.03)
z = np.arange(NZ + 1) * (np.pi / 256)
blk = mesh.BlockSpec(mesh._grid_vertices(x, y, z))
bnd = {(0, 0, 0): mesh._identity_conn(0, 0, 1, 3),
       (0, 0, 1): mesh._identity_conn(0, 0, 0, 3),
       (0, 1, 0): mesh.Dirichlet(0.0), (0, 1, 1): mesh.Dirichlet(0.0),
       (0, 2, 0): mesh._identity_conn(0, 2, 1, 3),
       (0, 2, 1): mesh._identity_conn(0, 2, 0, 3)}
dom = mesh.Domain([blk], bnd)
state, nu, _ = piso.reichardt_init(dom, 180.0, perturbation=0.1, seed=0)
dt = 0.3 * (2 * np.pi / 256) / np.abs(state.u).max()
print("n", dom.n, "dt", dt, "nu", nu)

systems = []
orig_bi = linalg.bicgstab_solve


def cap(tag):
    def f(pattern, data, b, x0=None, **kw):
        systems.append((tag, pattern, data.copy(), np.array(b),
                        None if x0 is None else np.array(x0)))
        return orig_bi(pattern, data, b, x0=x0, **kw)
    return f


piso.bicgstab_solve = cap("fwd")
adjoint.bicgstab_solve = cap("adj")
ws = piso.PisoWorkspace(dom)
w = np.random.default_rng(0).standard_normal((dom.n, 3))
for k in range(3):
    src = piso.wall_forcing_source(dom, state.u, nu)
    cfg = piso.StepConfig(dt=dt, nu=nu, source=src, tol=1e-8)
    tape = piso.StepTape()
    state, dg = piso.piso_step(dom, state, cfg, ws, tape)
    g = adjoint.backward_step(dom, tape, adjoint.GradState(
        u=w, p=np.zeros(dom.n)), tol=1e-8)
    print("step", k, "ref mom", dg.momentum_iterations, "adj", g.solve_iterations)
systems = systems[-6:]   # last step: 3 fwd + 3 adj


def bicgstab(A, b, x0, tol, M):
    x = np.zeros_like(b) if x0 is None else x0.copy()
    tol_abs = tol * np.linalg.norm(b)
    r = b - A @ x
    if np.linalg.norm(r) <= tol_abs:
        return 0
    rhat = r.copy()
    rho = al = om = 1.0
    v = np.zeros_like(b); p = np.zeros_like(b)
    for it in range(1, 500):
        rn = rhat @ r
        beta = (rn / rho) * (al / om)
        p = r + beta * (p - om * v)
        ph = M(p); v = A @ ph
        al = rn / (rhat @ v)
        s = r - al * v
        if np.linalg.norm(s) <= tol_abs:
            return it - 0.5
        sh = M(s); t = A @ sh
        om = (t @ s) / (t @ t)
        x = x + al * ph + om * sh
        r = s - om * t
        if np.linalg.norm(r) <= tol_abs:
            return it
        rho = rn
    return 999


for tag, pat, data, b, x0 in systems:
    A = sp.csr_matrix((data, pat.indices, pat.indptr), shape=(pat.n, pat.n))
    dg = A.diagonal()
    if tag == "adj":
        A = A.T.tocsr()
    n = pat.n
    # y-line tridiagonal part
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [dg]
    for s in (0, 1):
        nb = dom.nbr[1, s]
        ok = nb >= 0
        rows.append(np.nonzero(ok)[0]); cols.append(nb[ok])
        vals.append(np.asarray(A[np.nonzero(ok)[0], nb[ok]]).ravel())
    T = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows),
                                              np.concatenate(cols))),
                      shape=(n, n))
    lu = spla.splu(T)
    ilu = pat.factorize(data) if tag == "fwd" else None
    res = {"none": bicgstab(A, b, x0, 1e-8, lambda v: v),
           "jacobi": bicgstab(A, b, x0, 1e-8, lambda v: v / dg),
           "yline": bicgstab(A, b, x0, 1e-8, lambda v: lu.solve(v))}
    if ilu is not None:
        res["ilu0(ref)"] = bicgstab(A, b, x0, 1e-8, ilu.apply)
    print(tag, res)
