"""CPU oracle of the differentiable PISO step -- TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference algorithm (``pisoflow``,
/root/reference/pkg/src/pisoflow = S/) used as the checker for the CUDA
path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / reference legs may import it; the product never does.

Parity is PINNED: tests/test_oracle_golden.py checks every function here
against golden vectors produced by the reference itself
(tests/golden/make_golden.py).

Representation: matrices on the cell-adjacency pattern are (2d+1, n)
stencils (row 0 diagonal, row 1 + 2a + s the coupling across face (a, s)),
vector fields are (n, d) as in the reference.  The domain is duck-typed:
any object with the reference Domain's host arrays (``nbr``, ``nbr_ax``,
``nbr_sign``, ``jac``, ``tmat``, ``alpha``, ``bfaces``) works -- the
reference's own Domain or this repository's.

Linear solves are EXACT by default (sparse LU, the pressure pinned and
projected to zero mean): the reference's iterative solves converge to the
same discrete solutions within their tolerance, so an exact oracle is the
sharpest target.  ``cg`` / ``bicgstab`` restate the reference's Krylov
recurrences (S/linalg.py:136-212) for iteration-level checks with the
Jacobi preconditioner the GPU uses.

Scope: orthogonal grids (alpha diagonal), which covers every BASELINE
configuration; the lagged non-orthogonal fluxes are not restated here.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


# ---------------------------------------------------------------------------
# topology helpers


def faces(dom):
    """Yield (f, a, s, nsign, nb, ax, sign) for every face direction, with
    nb (n,) the neighbour (-1 at boundaries), ax/sign the neighbour's axis
    and orientation for my axis a (S/mesh.py:451-458)."""
    d = dom.dim
    for a in range(d):
        for s in (0, 1):
            nb = dom.nbr[a, s]
            ax = dom.nbr_ax[a, s, :, a].astype(np.int64)
            sg = dom.nbr_sign[a, s, :, a].astype(np.float64)
            yield 2 * a + s, a, s, (1.0 if s else -1.0), nb, ax, sg


def alpha_diag(dom):
    d = dom.dim
    return dom.alpha[:, np.arange(d), np.arange(d)]        # (n, d)


def boundary_entries(dom):
    """Flat per-entry arrays over dom.bfaces (reference order)."""
    out = []
    for f in dom.bfaces:
        out.append(dict(cells=f.cells, axis=f.axis, side=f.side,
                        nsign=f.nsign, kind=f.kind, jac=f.face_jac,
                        trow=f.face_t[:, f.axis, :],
                        alpha=f.face_alpha[:, f.axis, f.axis], m=f.m))
    return out


def flux(dom, u):
    """U^a = J (T u)_a  (S/piso.py:123-125)."""
    return dom.jac[:, None] * np.einsum("naj,nj->na", dom.tmat, u)


def stencil_matvec(dom, st, x, transpose=False):
    """y = A x for a stencil (S/_kernels_c.pyx:52-63 on the pattern)."""
    y = st[0] * x
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        if not transpose:
            y[ok] += st[1 + f][ok] * x[nb[ok]]
        else:
            # entry (i, nb) of A contributes A[i, nb] x_i to row nb
            np.add.at(y, nb[ok], st[1 + f][ok] * x[ok])
    return y


def to_csr(dom, st):
    n = dom.n
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [st[0]]
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        rows.append(np.nonzero(ok)[0])
        cols.append(nb[ok])
        vals.append(st[1 + f][ok])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                 np.concatenate(cols))),
                         shape=(n, n))


# ---------------------------------------------------------------------------
# forward building blocks


def assemble_momentum(dom, u, nu, dt):
    """Advection-diffusion stencil, rows / J (S/piso.py:293-319)."""
    n, d = dom.n, dom.dim
    U = flux(dom, u)
    invj = 1.0 / dom.jac
    ad = alpha_diag(dom)
    st = np.zeros((2 * d + 1, n))
    diag = np.full(n, 1.0 / dt)
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        safe = np.maximum(nb, 0)
        unb = sg * U[safe, ax]
        fmean = 0.5 * (U[:, a] + unb)
        adv = 0.5 * ns * fmean * invj
        visc = 0.5 * (nu * ad[:, a] + nu * ad[safe, ax]) * invj
        st[1 + f] = np.where(ok, adv - visc, 0.0)
        diag += np.where(ok, adv + visc, 0.0)
    for e in boundary_entries(dom):
        if e["kind"] == "dirichlet":
            diag[e["cells"]] += 2.0 * nu * e["alpha"] / dom.jac[e["cells"]]
    st[0] = diag
    return st


def momentum_rhs(dom, u, bc, nu, dt, src):
    """u/dt + S + boundary terms (S/piso.py:356-372, orthogonal)."""
    rhs = u / dt + src
    invj = 1.0 / dom.jac
    for e, ub in zip(boundary_entries(dom), bc):
        c = e["cells"]
        uflux = e["jac"] * np.einsum("mj,mj->m", e["trow"], ub)
        if e["kind"] == "dirichlet":
            w = (2.0 * nu * e["alpha"] - uflux * e["nsign"]) * invj[c]
        else:
            w = -uflux * e["nsign"] * invj[c]
        rhs[c] += ub * w[:, None]
    return rhs


def assemble_pressure(dom, a_inv):
    """P stencil: face means of alpha_aa A^-1, zero row sums
    (S/piso.py:395-412)."""
    n, d = dom.n, dom.dim
    ad = alpha_diag(dom)
    st = np.zeros((2 * d + 1, n))
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        safe = np.maximum(nb, 0)
        pf = 0.5 * (ad[:, a] * a_inv + ad[safe, ax] * a_inv[safe])
        st[1 + f] = np.where(ok, pf, 0.0)
        st[0] -= np.where(ok, pf, 0.0)
    return st


def divergence_rhs(dom, h, bc):
    """xi-space flux divergence with boundary fluxes (S/piso.py:415-428)."""
    U = flux(dom, h)
    b = np.zeros(dom.n)
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        safe = np.maximum(nb, 0)
        b += ns * np.where(ok, 0.5 * (U[:, a] + sg * U[safe, ax]), 0.0)
    for e, ub in zip(boundary_entries(dom), bc):
        np.add.at(b, e["cells"],
                  e["nsign"] * e["jac"] * np.einsum("mj,mj->m", e["trow"], ub))
    return b


def mirror_grad(dom, p):
    """wide_grad(p, 'mirror') (S/piso.py:172-209)."""
    d = dom.dim
    g = np.empty((dom.n, d))
    for a in range(d):
        hi, lo = dom.nbr[a, 1], dom.nbr[a, 0]
        vhi = np.where(hi >= 0, p[np.maximum(hi, 0)], p)
        vlo = np.where(lo >= 0, p[np.maximum(lo, 0)], p)
        g[:, a] = 0.5 * (vhi - vlo)
    return g


def correct_velocity(dom, h, p, a_inv):
    """u = h - A^-1 T^t grad(p) (S/piso.py:452-455)."""
    return h - a_inv[:, None] * np.einsum("nji,nj->ni", dom.tmat,
                                          mirror_grad(dom, p))


def advective_outflow_update(dom, u, bc, dt):
    """Relax + rebalance outflow faces (S/piso.py:467-509)."""
    ents = boundary_entries(dom)
    bc = [b.copy() for b in bc]
    if not any(e["kind"] == "advective_outflow" for e in ents):
        return bc, 1.0

    def face_flux(e, ub):
        return float(np.sum(e["nsign"] * e["jac"]
                            * np.einsum("mj,mj->m", e["trow"], ub)))

    fixed = sum(face_flux(e, b) for e, b in zip(ents, bc)
                if e["kind"] == "dirichlet")
    out = 0.0
    for k, e in enumerate(ents):
        if e["kind"] != "advective_outflow":
            continue
        speed = np.einsum("mj,mj->m", e["trow"], bc[k])
        a = np.maximum(2.0 * dt * speed * e["nsign"], 0.0)
        bc[k] = (bc[k] + a[:, None] * u[e["cells"]]) / (1.0 + a)[:, None]
        out += face_flux(e, bc[k])
    if abs(out) < 1e-13 * max(1.0, abs(fixed)):
        if abs(fixed) <= 1e-12:
            return bc, 1.0
        area = sum(float(e["jac"].sum()) for e in ents
                   if e["kind"] == "advective_outflow")
        c = -fixed / area
        for k, e in enumerate(ents):
            if e["kind"] == "advective_outflow":
                t = e["trow"]
                bc[k] = c * e["nsign"] * (t / np.einsum("mj,mj->m", t,
                                                        t)[:, None])
        return bc, 1.0
    scale = -fixed / out
    for k, e in enumerate(ents):
        if e["kind"] == "advective_outflow":
            bc[k] = bc[k] * scale
    return bc, scale


# ---------------------------------------------------------------------------
# linear solves


def solve_exact(dom, st, b, transpose=False):
    A = to_csr(dom, st)
    if transpose:
        A = A.T.tocsc()
    return spla.spsolve(A.tocsc(), b)


def solve_pressure_exact(dom, k_st, b):
    """Zero-mean solution of the singular K p = b - mean(b)."""
    K = to_csr(dom, k_st).tolil()
    rhs = b - b.mean()
    K[0, :] = 0.0
    K[0, 0] = 1.0
    rhs = rhs.copy()
    rhs[0] = 0.0
    x = spla.spsolve(K.tocsc(), rhs)
    return x - x.mean()


def cg(dom, st, b, x0=None, tol=1e-8, maxiter=None, precond="jacobi",
       zero_mean=True, variant="classic"):
    """Restatement of cg_solve/_cg_core/_run_with_fallback
    (S/linalg.py:136-170, 215-273).  Returns (x, converged, iterations).
    variant="single": the product's single-reduction form of the same
    iteration (Chronopoulos & Gear: w = K z carried alongside, the step
    length from r.z and z.w of one pass; same iterates in exact
    arithmetic), checked against the classic loop."""
    n = dom.n
    if maxiter is None:
        maxiter = max(200, 40 * int(round(n ** 0.5)))
    b = b - b.mean() if zero_mean else b.copy()
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), True, 0
    tol_abs = tol * bnorm

    def core(x, pc, mi):
        def M(r):
            z = r / st[0] if pc else r.copy()
            return z - z.mean() if zero_mean else z
        r = b - stencil_matvec(dom, st, x)
        if zero_mean:
            r -= r.mean()
        res = np.linalg.norm(r)
        if res <= tol_abs:
            return x, True, 0
        z = M(r)
        p = z.copy()
        rz = float(r @ z)
        for it in range(1, mi + 1):
            q = stencil_matvec(dom, st, p)
            pq = float(p @ q)
            if not np.isfinite(pq) or abs(pq) < np.finfo(float).tiny:
                return x, False, it
            al = rz / pq
            x = x + al * p
            r = r - al * q
            if np.linalg.norm(r) <= tol_abs:
                if zero_mean:
                    x = x - x.mean()
                return x, True, it
            z = M(r)
            rzn = float(r @ z)
            if not np.isfinite(rzn) or rz == 0.0:
                return x, False, it
            p = z + (rzn / rz) * p
            rz = rzn
        return x, False, mi

    def core_single(x, pc, mi):
        def M(r):
            z = r / st[0] if pc else r.copy()
            return z - z.mean() if zero_mean else z

        def K(v):
            return stencil_matvec(dom, st, v)
        r = b - K(x)
        if zero_mean:
            r -= r.mean()
        if np.linalg.norm(r) <= tol_abs:
            return x, True, 0
        z = M(r)
        w = K(z)
        g, d = float(r @ z), float(z @ w)
        if not np.isfinite(d) or abs(d) < np.finfo(float).tiny:
            return x, False, 0
        al, be = g / d, 0.0
        p, s_ = np.zeros(n), np.zeros(n)
        for it in range(1, mi + 1):
            p = z + be * p
            s_ = w + be * s_
            x = x + al * p
            r = r - al * s_
            z = M(r)
            w = K(z)
            # one reduction: |r|, r.z, z.w
            res, gn, d = np.linalg.norm(r), float(r @ z), float(z @ w)
            if res <= tol_abs:
                if zero_mean:
                    x = x - x.mean()
                return x, True, it
            if it >= mi:
                break
            if not np.isfinite(gn) or g == 0.0:
                return x, False, it
            be = gn / g
            pap = d - be * gn / al
            if not np.isfinite(pap) or abs(pap) < np.finfo(float).tiny:
                return x, False, it
            al, g = gn / pap, gn
        return x, False, mi

    if variant == "single":
        core = core_single
    x = np.zeros(n) if x0 is None else x0.copy()
    x, ok, it = core(x, precond is not None, maxiter)
    if ok:
        ok = np.linalg.norm(b - stencil_matvec(dom, st, x)) <= 10 * tol_abs
    if not ok and precond is not None:
        x, ok, it2 = core(np.zeros(n), False, 2 * maxiter)
        it += it2
    return x, ok, it


def bicgstab(dom, st, b, x0=None, tol=1e-8, maxiter=None, precond="jacobi",
             transpose=False):
    """Restatement of _bicgstab_core (S/linalg.py:173-212) with the same
    wrapper semantics.  Returns (x, converged, iterations).  precond:
    "jacobi", or "neumann2" -- the product's two-sweep Jacobi polynomial
    M^-1 = D^-1 - D^-1 N D^-1 (N = A - D), checked here as a plain
    right preconditioner (the product keeps the iterate as x0 + M^-1 z,
    which is the same sequence of iterates)."""
    n = dom.n
    if maxiter is None:
        maxiter = max(200, 40 * int(round(n ** 0.5)))
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), True, 0
    tol_abs = tol * bnorm
    tiny = np.finfo(float).tiny

    def A(v):
        return stencil_matvec(dom, st, v, transpose=transpose)

    def core(x, pc, mi):
        def M(v):
            if not pc:
                return v
            g = v / st[0]
            if precond != "neumann2":
                return g
            return g - (A(g) - st[0] * g) / st[0]
        r = b - A(x)
        if np.linalg.norm(r) <= tol_abs:
            return x, True, 0
        rh = r.copy()
        rho = alpha = omega = 1.0
        v = np.zeros(n)
        p = np.zeros(n)
        for it in range(1, mi + 1):
            rho_n = float(rh @ r)
            if abs(rho_n) < tiny or abs(omega) < tiny:
                return x, False, it
            beta = (rho_n / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
            ph = M(p)
            v = A(ph)
            den = float(rh @ v)
            if abs(den) < tiny:
                return x, False, it
            alpha = rho_n / den
            s = r - alpha * v
            if np.linalg.norm(s) <= tol_abs:
                return x + alpha * ph, True, it
            sh = M(s)
            t = A(sh)
            tt = float(t @ t)
            if tt < tiny:
                return x, False, it
            omega = float(t @ s) / tt
            x = x + alpha * ph + omega * sh
            r = s - omega * t
            if np.linalg.norm(r) <= tol_abs:
                return x, True, it
            rho = rho_n
        return x, False, mi

    x = np.zeros(n) if x0 is None else x0.copy()
    x, ok, it = core(x, precond is not None, maxiter)
    if ok:
        ok = np.linalg.norm(b - A(x)) <= 10 * tol_abs
    if not ok and precond is not None:
        x, ok, it2 = core(np.zeros(n), False, 2 * maxiter)
        it += it2
    return x, ok, it


# ---------------------------------------------------------------------------
# the step and its adjoint


@dataclass
class Tape:
    dt: float
    nu: float
    u_n: np.ndarray
    bc: list
    C: np.ndarray
    rhs: np.ndarray
    u_star: np.ndarray
    K: np.ndarray
    correctors: list = field(default_factory=list)  # (u_hin, h, p)


def resolve_source(dom, source):
    n, d = dom.n, dom.dim
    if source is None:
        return np.zeros((n, d))
    s = np.asarray(source, dtype=np.float64)
    return np.tile(s, (n, 1)) if s.shape == (d,) else s.copy()


def piso_step(dom, u, p, bc, dt, nu, source=None, n_correctors=2,
              solver="exact", tol=1e-12):
    """One PISO step (S/piso.py:561-654) on an orthogonal grid.
    Returns (u, p, bc, tape, diagnostics dict)."""
    src = resolve_source(dom, source)
    bc, scale = advective_outflow_update(dom, u, bc, dt)
    C = assemble_momentum(dom, u, nu, dt)
    rhs = momentum_rhs(dom, u, bc, nu, dt, src)
    d = dom.dim
    u_star = np.empty_like(u)
    it_m = 0
    for c in range(d):
        if solver == "exact":
            u_star[:, c] = solve_exact(dom, C, rhs[:, c])
        else:
            u_star[:, c], ok, k = bicgstab(dom, C, rhs[:, c], tol=tol)
            it_m += k
    a_inv = 1.0 / C[0]
    K = -assemble_pressure(dom, a_inv)
    tape = Tape(dt, nu, u.copy(), [b.copy() for b in bc], C, rhs, u_star, K)
    u_cur = u_star
    it_p = 0
    for m in range(n_correctors):
        hu = stencil_matvec_off(dom, C, u_cur)
        h = a_inv[:, None] * (rhs - hu)
        b0 = divergence_rhs(dom, h, bc)
        if solver == "exact":
            p = solve_pressure_exact(dom, K, -b0)
        else:
            p, ok, k = cg(dom, K, -b0, tol=tol)
            it_p += k
        tape.correctors.append((u_cur, h, p))
        u_cur = correct_velocity(dom, h, p, a_inv)
    div = divergence_rhs(dom, u_cur, bc) / dom.jac
    return u_cur, p, bc, tape, dict(advout_scale=scale,
                                    div_wide_max=float(np.abs(div).max()),
                                    momentum_iterations=it_m,
                                    pressure_iterations=it_p)


def stencil_matvec_off(dom, st, u):
    """H u = (C - A) u per component."""
    out = np.zeros_like(u)
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        out[ok] += st[1 + f][ok][:, None] * u[nb[ok]]
    return out


def _scatter_nb(acc, dom, f_vals_by_face, comp_by_face=None):
    """acc[nb, comp] += vals for each face (np.add.at transposes)."""
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        vals = f_vals_by_face[f]
        if comp_by_face is None:
            np.add.at(acc, nb[ok], vals[ok])
        else:
            np.add.at(acc, (nb[ok], ax[ok]), (sg * vals)[ok])


def backward_step(dom, tape, cot_u, cot_p=None, path="full",
                  solver="exact", tol=1e-12):
    """Reverse of one step (S/adjoint.py:412-506), orthogonal grids.
    Returns dict(u, nu, source, bc)."""
    n, d = dom.n, dom.dim
    C, K = tape.C, tape.K
    A = C[0]
    a_inv = 1.0 / A
    ad = alpha_diag(dom)
    ents = boundary_entries(dom)
    press = path in ("full", "p_only")
    adv = path in ("full", "adv_only")
    dC = np.zeros_like(C)
    dA = np.zeros(n)
    dPf = np.zeros((2 * d, n))       # y_i (p_nb - p_i) per face
    g_rhs = np.zeros((n, d))
    dbc = [np.zeros((e["m"], d)) for e in ents]
    cu = np.array(cot_u, dtype=np.float64)
    for m in reversed(range(len(tape.correctors))):
        u_hin, h, p = tape.correctors[m]
        # correct_velocity (S/adjoint.py:78-91)
        ep = np.einsum("nji,nj->ni", dom.tmat, mirror_grad(dom, p))
        dA += np.einsum("ni,ni->n", cu, ep) * a_inv ** 2
        cot_gp = np.einsum("nji,ni->nj", dom.tmat, -a_inv[:, None] * cu)
        dp = np.zeros(n)
        for a in range(d):
            hi, lo = dom.nbr[a, 1], dom.nbr[a, 0]
            c = 0.5 * cot_gp[:, a]
            np.add.at(dp, hi[hi >= 0], c[hi >= 0])
            np.add.at(dp, lo[lo >= 0], -c[lo >= 0])
            dp += np.where(hi < 0, c, 0.0) - np.where(lo < 0, c, 0.0)
        cot_pm = dp + (cot_p if (m == len(tape.correctors) - 1
                                 and cot_p is not None) else 0.0)
        g_h = cu.copy()
        if press:
            chat = cot_pm - cot_pm.mean()
            if solver == "exact":
                y = solve_pressure_exact(dom, K, chat)
            else:
                y, ok, k = cg(dom, K, chat, tol=tol)
            for f, a, s, ns, nb, ax, sg in faces(dom):
                ok = nb >= 0
                dPf[f] += np.where(ok, y * (p[np.maximum(nb, 0)] - p), 0.0)
            cot_b = -y
            # _adj_divergence_rhs (S/adjoint.py:137-153)
            gflux = np.zeros((n, d))
            vals = {}
            for f, a, s, ns, nb, ax, sg in faces(dom):
                cf = 0.5 * ns * np.where(nb >= 0, cot_b, 0.0)
                gflux[:, a] += cf
                vals[f] = cf
            _scatter_nb(gflux, dom, vals, comp_by_face=True)
            g_h += dom.jac[:, None] * np.einsum("naj,na->nj", dom.tmat, gflux)
            for k, e in enumerate(ents):
                coef = e["nsign"] * e["jac"] * cot_b[e["cells"]]
                dbc[k] += coef[:, None] * e["trow"]
        # h stage (S/adjoint.py:477-487)
        dA += -a_inv * np.einsum("nc,nc->n", g_h, h)
        grhs = a_inv[:, None] * g_h
        g_rhs += grhs
        cot_hu = -grhs
        cu_new = np.zeros((n, d))
        for f, a, s, ns, nb, ax, sg in faces(dom):
            ok = nb >= 0
            safe = np.maximum(nb, 0)
            dC[1 + f] += np.where(ok, np.einsum("nc,nc->n", cot_hu,
                                                u_hin[safe]), 0.0)
            np.add.at(cu_new, nb[ok], C[1 + f][ok][:, None] * cot_hu[ok])
        cu = cu_new
    if press:
        # backward_pressure_matrix (S/adjoint.py:116-134)
        g = np.zeros(n)
        for f, a, s, ns, nb, ax, sg in faces(dom):
            ok = nb >= 0
            g += 0.5 * dPf[f] * ad[:, a]
            np.add.at(g, nb[ok], (0.5 * dPf[f] * ad[np.maximum(nb, 0),
                                                     ax])[ok])
        dA += -a_inv ** 2 * g
    dC[0] += dA
    # predictor (S/adjoint.py:343-405)
    grhs = g_rhs.copy()
    if adv:
        y = np.zeros((n, d))
        for c in range(d):
            if solver == "exact":
                y[:, c] = solve_exact(dom, C, cu[:, c], transpose=True)
            else:
                y[:, c], ok, k = bicgstab(dom, C, cu[:, c], tol=tol,
                                          transpose=True)
        us = tape.u_star
        dC[0] += np.einsum("nc,nc->n", -y, us)
        for f, a, s, ns, nb, ax, sg in faces(dom):
            ok = nb >= 0
            dC[1 + f] += np.where(ok, np.einsum(
                "nc,nc->n", -y, us[np.maximum(nb, 0)]), 0.0)
        grhs += y
    du = grhs / tape.dt
    dnu = 0.0
    invj = 1.0 / dom.jac
    nu = tape.nu
    for k, (e, ub) in enumerate(zip(ents, tape.bc)):
        c = e["cells"]
        cr = grhs[c]
        uflux = e["jac"] * np.einsum("mj,mj->m", e["trow"], ub)
        crub = np.einsum("mj,mj->m", cr, ub)
        if e["kind"] == "dirichlet":
            coef = (2.0 * nu * e["alpha"] - uflux * e["nsign"]) * invj[c]
            dnu += float(np.sum(crub * 2.0 * e["alpha"] * invj[c]))
        else:
            coef = -uflux * e["nsign"] * invj[c]
        cot_uf = -e["nsign"] * invj[c] * crub
        dbc[k] += cr * coef[:, None] + (cot_uf * e["jac"])[:, None] * e["trow"]
    # assembly adjoint (S/adjoint.py:307-340)
    gflux = np.zeros((n, d))
    vals = {}
    for f, a, s, ns, nb, ax, sg in faces(dom):
        ok = nb >= 0
        safe = np.maximum(nb, 0)
        cot_off = np.where(ok, dC[1 + f], 0.0)
        cd = np.where(ok, dC[0], 0.0)
        cadv = cot_off + cd
        cvis = cd - cot_off
        dnu += float(np.sum(cvis * 0.5 * (ad[:, a] + np.where(
            ok, ad[safe, ax], 0.0)) * invj))
        cfm = 0.5 * ns * invj * cadv
        gflux[:, a] += 0.5 * cfm
        vals[f] = 0.5 * cfm
    _scatter_nb(gflux, dom, vals, comp_by_face=True)
    for e in ents:
        if e["kind"] == "dirichlet":
            c = e["cells"]
            dnu += float(np.sum(dC[0][c] * 2.0 * e["alpha"] * invj[c]))
    du += dom.jac[:, None] * np.einsum("naj,na->nj", dom.tmat, gflux)
    return dict(u=du, nu=dnu, source=grhs, bc=dbc)


def rollout(dom, u0, bc0, dt, nu, steps, source=None, n_correctors=2,
            solver="exact", tol=1e-12):
    u, p, bc = u0.copy(), np.zeros(dom.n), [b.copy() for b in bc0]
    tapes, outs = [], []
    for _ in range(steps):
        u, p, bc, tape, dg = piso_step(dom, u, p, bc, dt, nu, source,
                                       n_correctors, solver, tol)
        tapes.append(tape)
        outs.append((u.copy(), p.copy(), [b.copy() for b in bc], dg))
    return tapes, outs


def backward_rollout(dom, tapes, cot_u_last, cot_p_last=None, path="full",
                     solver="exact", tol=1e-12):
    """Cotangent on the last state only (S/adjoint.py:509-539)."""
    cu = np.array(cot_u_last, dtype=np.float64)
    total_nu = 0.0
    total_src = np.zeros_like(cu)
    total_bc = None
    for k in reversed(range(len(tapes))):
        g = backward_step(dom, tapes[k], cu,
                          cot_p_last if k == len(tapes) - 1 else None,
                          path, solver, tol)
        total_nu += g["nu"]
        total_src += g["source"]
        total_bc = g["bc"] if total_bc is None else [
            a + b for a, b in zip(total_bc, g["bc"])]
        cu = g["u"]
    return dict(u=cu, nu=total_nu, source=total_src, bc=total_bc)
