"""Discrete adjoint of the PISO step on device (mirror of S/adjoint.py).

``backward_step`` / ``backward_rollout`` keep the reference's signatures,
gradient-path gating (``GradientPath``), stage labels and ``GradState``
(S/adjoint.py:28-66, 412-539).  Every stage is a kernel of
``libpisob200.so``; transposes are gathers over the neighbour relation, so
the result is bitwise reproducible.

Stage map (orthogonal grids):

=============================  ===========================  ==========================
reverse of                     reference                    kernel entry
=============================  ===========================  ==========================
correct_velocity               S/adjoint.py:78-91           pf_bwd_correct_velocity
pressure solve (adjoint CG)    S/adjoint.py:94-113          pf_cg_solve + pf_bwd_pressure_outer
pressure assembly              S/adjoint.py:116-134         pf_bwd_pressure_matrix
divergence_rhs                 S/adjoint.py:137-153         pf_adj_divergence_rhs
h stage                        S/adjoint.py:477-487         pf_bwd_h_stage
momentum solve (adjoint BiCG)  S/adjoint.py:369-380         pf_bicgstab_solve(A^t) + pf_bwd_momentum_outer
momentum_rhs                   S/adjoint.py:236-268         pf_adj_momentum_rhs
assemble_momentum              S/adjoint.py:307-340         pf_adj_assemble_momentum
=============================  ===========================  ==========================
"""

from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _lib
from .linalg import bicgstab_solve, cg_solve
from .piso import F64, bc_views, scalar_field, soa


class GradientPath(Enum):
    FULL = "full"
    ADV_ONLY = "adv_only"
    P_ONLY = "p_only"
    NONE = "none"

    @classmethod
    def parse(cls, name):
        for p in cls:
            if p.value == str(name).strip().lower():
                return p
        raise ValueError(f"unknown gradient path {name!r}; choose from "
                         + ", ".join(p.value for p in cls))

    @property
    def pressure_solve(self):
        return self in (GradientPath.FULL, GradientPath.P_ONLY)

    @property
    def advection_solve(self):
        return self in (GradientPath.FULL, GradientPath.ADV_ONLY)


@dataclass
class GradState:
    """Cotangents shaped like the state fields (S/adjoint.py:51-66)."""
    u: object
    p: object
    nu: float = 0.0
    source: object = None
    bc: list = None
    solve_iterations: int = 0
    reports: list = None     # SolverReports of the adjoint solves

    @classmethod
    def zeros(cls, domain, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if device is None else torch.device(device)
        n, d = domain.n, domain.dim
        plan = domain.device_plan(dev)
        bc = torch.zeros((d, plan.m), dtype=F64, device=dev) if plan.m \
            else None
        return cls(u=torch.zeros((d, n), dtype=F64, device=dev).t(),
                   p=torch.zeros(n, dtype=F64, device=dev), nu=0.0,
                   source=torch.zeros((d, n), dtype=F64, device=dev).t(),
                   bc=bc_views(plan, bc))


def backward_step(domain, tape, cot, path=GradientPath.FULL, tol=None,
                  maxiter=None):
    """Chain the backward kernels through one recorded step
    (S/adjoint.py:412-506)."""
    if tape is None or tape.u_n is None:
        raise ValueError("backward_step needs a recorded tape")
    if isinstance(path, str):
        path = GradientPath.parse(path)
    dev = tape.c_data.device
    plan = domain.device_plan(dev)
    n, d = domain.n, domain.dim
    hs = plan.stream
    C, K = tape.c_data, tape.k_data
    n_corr = len(tape.correctors)
    reports = []

    # first writers store (overwrite flag) instead of the kernels adding to
    # zero-filled accumulators; slab plans keep the fill (ghost planes are
    # not written by the owned-range kernels)
    ow = 0 if plan.slab else 1
    alloc = torch.zeros if plan.slab else torch.empty
    dC = alloc((2 * d + 1, n), dtype=F64, device=dev)
    dA = dC[0]                       # dC[diag] += dA (S/adjoint.py:492)
    dKf = alloc((2 * d, n), dtype=F64, device=dev)
    g_rhs = alloc((d, n), dtype=F64, device=dev)
    dbc = torch.zeros((d, plan.m), dtype=F64, device=dev) if plan.m else None
    dnu = torch.zeros(1, dtype=F64, device=dev)

    cu = soa(cot.u, n, d, dev).clone()
    cp_out = None if cot.p is None else scalar_field(cot.p, n, dev)
    cot_p = torch.empty(n, dtype=F64, device=dev)
    cu_next = torch.empty((d, n), dtype=F64, device=dev)
    pressure_done = False

    for m in reversed(range(n_corr)):
        corr = tape.correctors[m]
        p_m = corr.p_iters[-1]
        first = ow if m == n_corr - 1 else 0
        _lib.call("pf_bwd_correct_velocity", plan.handle, _lib.ptr(p_m),
                  _lib.ptr(C), _lib.ptr(cu), _lib.ptr(dA), _lib.ptr(cot_p),
                  _lib.ptr(cp_out if m == n_corr - 1 else None), first,
                  _lib.ptr(plan.workspace), hs)
        g_h = cu                     # dh = cu; the divergence adjoint adds
        n_it = len(corr.p_iters)
        if path.pressure_solve and not plan.cell_cross:
            # orthogonal grids: the lagged-cross adjoint that would feed the
            # earlier outer iterates is identically zero, so only the last
            # iterate carries a cotangent
            it = n_it - 1
            y, rep = cg_solve(plan, K, cot_p, tol=tol, maxiter=maxiter,
                              zero_mean=True, stage="adjoint_pressure")
            reports.append(rep)
            _lib.call("pf_bwd_pressure_outer", plan.handle, _lib.ptr(y),
                      _lib.ptr(corr.p_iters[it]), _lib.ptr(dKf),
                      0 if pressure_done else ow, hs)
            pressure_done = True
            # forward solved (-P) p = proj(-b): db = -y
            _lib.call("pf_adj_divergence_rhs", plan.handle, _lib.ptr(y),
                      -1.0, _lib.ptr(g_h), _lib.ptr(dbc), hs)
        elif path.pressure_solve:
            # S/adjoint.py:456-470: reversed outer iterates, each adjoint
            # solve feeding the previous iterate through the cross flux
            cot_b0 = torch.zeros(n, dtype=F64, device=dev)
            cp_it = cot_p
            for it in reversed(range(n_it)):
                y, rep = cg_solve(plan, K, cp_it, tol=tol, maxiter=maxiter,
                                  zero_mean=True, stage="adjoint_pressure")
                if rep.iterations or rep.residual:
                    reports.append(rep)
                _lib.call("pf_bwd_pressure_outer", plan.handle, _lib.ptr(y),
                          _lib.ptr(corr.p_iters[it]), _lib.ptr(dKf),
                          0 if pressure_done else ow, hs)
                pressure_done = True
                _lib.call("pf_axpy", plan.handle, -1.0, _lib.ptr(y),
                          _lib.ptr(cot_b0), n, hs)
                if it > 0:
                    nxt = torch.empty(n, dtype=F64, device=dev)
                    # cot of the cross flux = -db = y
                    _lib.call("pf_adj_pressure_cross", plan.handle,
                              _lib.ptr(C), _lib.ptr(corr.p_iters[it - 1]),
                              _lib.ptr(y), 1.0, _lib.ptr(dA), _lib.ptr(nxt),
                              _lib.ptr(plan.workspace), hs)
                    cp_it = nxt
            pressure_done = True
            _lib.call("pf_adj_divergence_rhs", plan.handle, _lib.ptr(cot_b0),
                      1.0, _lib.ptr(g_h), _lib.ptr(dbc), hs)
        _lib.call("pf_bwd_h_stage", plan.handle, _lib.ptr(C), _lib.ptr(g_h),
                  _lib.ptr(soa(corr.h, n, d, dev)),
                  _lib.ptr(soa(corr.u_hin, n, d, dev)), _lib.ptr(dA),
                  _lib.ptr(g_rhs), _lib.ptr(dC), _lib.ptr(cu_next), first,
                  _lib.ptr(plan.workspace), hs)
        cu, cu_next = cu_next, cu

    if pressure_done:
        _lib.call("pf_bwd_pressure_matrix", plan.handle, _lib.ptr(C),
                  _lib.ptr(dKf), _lib.ptr(dA), hs)

    # predictor (S/adjoint.py:343-405)
    du_n = alloc((d, n), dtype=F64, device=dev)
    du_first = ow
    bcd = getattr(tape, "_bc_dm", None)
    if bcd is None and plan.m:
        from .piso import bc_soa
        bcd = bc_soa(plan, tape.bc, d)
    n_outer = len(tape.mom_iters)
    stages = [f"adjoint_momentum[{c}]" for c in range(d)]
    # on orthogonal grids the cross-flux adjoint feeding earlier outer
    # iterates vanishes: only the last iterate carries a cotangent
    its = range(n_outer - 1, -1, -1) if plan.cell_cross else [n_outer - 1]
    dsource = None
    cot_us = cu
    for it in its:
        grhs = None
        if path.advection_solve:
            y, reps = bicgstab_solve(plan, C, cot_us, tol=tol,
                                     maxiter=maxiter, transpose=True,
                                     stages=stages)
            reports.extend(r for r in reps if r.iterations or r.residual)
            u_star = soa(tape.mom_iters[it], n, d, dev)
            _lib.call("pf_bwd_momentum_outer", plan.handle, _lib.ptr(y),
                      _lib.ptr(u_star), _lib.ptr(dC), hs)
            grhs = y
        if grhs is None:
            grhs = torch.zeros((d, n), dtype=F64, device=dev)
        if it == n_outer - 1:
            grhs.add_(g_rhs)
        _lib.call("pf_adj_momentum_rhs", plan.handle, _lib.ptr(grhs),
                  _lib.ptr(bcd), float(tape.nu), float(tape.dt),
                  _lib.ptr(du_n), _lib.ptr(dbc), _lib.ptr(dnu), du_first,
                  _lib.ptr(plan.workspace), hs)
        du_first = 0
        dsource = grhs if dsource is None else dsource.add_(grhs)
        if plan.cell_cross:
            u_in = soa(tape.mom_inputs[it], n, d, dev)
            if it == 0:
                _lib.call("pf_adj_momentum_cross", plan.handle,
                          _lib.ptr(u_in), float(tape.nu), _lib.ptr(grhs),
                          _lib.ptr(du_n), 1, _lib.ptr(dnu),
                          _lib.ptr(plan.workspace), hs)
            else:
                nxt = torch.empty((d, n), dtype=F64, device=dev)
                _lib.call("pf_adj_momentum_cross", plan.handle,
                          _lib.ptr(u_in), float(tape.nu), _lib.ptr(grhs),
                          _lib.ptr(nxt), 0, _lib.ptr(dnu),
                          _lib.ptr(plan.workspace), hs)
                cot_us = nxt
    _lib.call("pf_adj_assemble_momentum", plan.handle, _lib.ptr(dC),
              float(tape.nu), _lib.ptr(du_n), _lib.ptr(dnu),
              _lib.ptr(plan.workspace), hs)
    iters = sum(r.iterations for r in reports)
    return GradState(u=du_n.t(), p=torch.zeros(n, dtype=F64, device=dev),
                     nu=float(dnu.item()), source=dsource.t(),
                     bc=bc_views(plan, dbc), solve_iterations=iters,
                     reports=reports)


# ---------------------------------------------------------------------------
# stage API (S/adjoint.py:78-205): the adjoint building blocks on their own.
# backward_step chains the same kernels; these wrappers expose them with the
# reference's arguments (per-cell device tensors; matrix cotangents in this
# package's stencil / face layout instead of CSR pattern values).


def backward_correct_velocity(domain, p, a_diag, cot_u):
    """Reverse of u = h - A^-1 T^t grad_xi(p) (S/adjoint.py:78-91).
    Returns (dA, dp, dh).  Kernel: pf_bwd_correct_velocity."""
    from .piso import _cdiag
    plan = domain.device_plan(cot_u.device)
    n, d = domain.n, domain.dim
    da = torch.zeros(n, dtype=F64, device=plan.device)
    dp = torch.empty(n, dtype=F64, device=plan.device)
    cu = soa(cot_u, n, d, plan.device)
    _lib.call("pf_bwd_correct_velocity", plan.handle,
              _lib.ptr(scalar_field(p, n, plan.device)),
              _lib.ptr(_cdiag(a_diag, n, plan.device)), _lib.ptr(cu),
              _lib.ptr(da), _lib.ptr(dp), _lib.ptr(None), 0,
              _lib.ptr(plan.workspace), plan.stream)
    return da, dp, cu.clone().t()


def _adj_divergence_rhs(domain, cot_b):
    """Adjoint of divergence_rhs in (h, bc) (S/adjoint.py:137-153).
    Returns (dh (n, d), [dbc (m, d) per boundary face])."""
    plan = domain.device_plan(cot_b.device)
    n, d = domain.n, domain.dim
    dh = torch.zeros((d, n), dtype=F64, device=plan.device)
    dbc = torch.zeros((d, plan.m), dtype=F64, device=plan.device) \
        if plan.m else None
    _lib.call("pf_adj_divergence_rhs", plan.handle,
              _lib.ptr(scalar_field(cot_b, n, plan.device)), 1.0,
              _lib.ptr(dh), _lib.ptr(dbc), plan.stream)
    return dh.t(), bc_views(plan, dbc)


def _adj_pressure_cross(domain, a_inv, p_prev, cot_out):
    """Adjoint of the lagged non-orthogonal pressure fluxes
    (S/adjoint.py:156-178).  Returns (dp_prev, d_ainv)."""
    from .piso import _cdiag
    plan = domain.device_plan(cot_out.device)
    n = domain.n
    dp = torch.zeros(n, dtype=F64, device=plan.device)
    if not plan.cell_cross:
        return dp, torch.zeros(n, dtype=F64, device=plan.device)
    ainv = scalar_field(a_inv, n, plan.device)
    a = 1.0 / ainv
    da = torch.zeros(n, dtype=F64, device=plan.device)
    _lib.call("pf_adj_pressure_cross", plan.handle,
              _lib.ptr(_cdiag(a, n, plan.device)),
              _lib.ptr(scalar_field(p_prev, n, plan.device)),
              _lib.ptr(scalar_field(cot_out, n, plan.device)), 1.0,
              _lib.ptr(da), _lib.ptr(dp), _lib.ptr(plan.workspace),
              plan.stream)
    # the kernel accumulates the cotangent of A; a_inv = 1 / A
    return dp, -da * a * a


def _adj_momentum_cross(domain, u_cross, nu, cot_out):
    """Adjoint of the lagged non-orthogonal viscous fluxes
    (S/adjoint.py:181-205).  Returns (du_cross (n, d), dnu)."""
    plan = domain.device_plan(cot_out.device)
    n, d = domain.n, domain.dim
    du = torch.zeros((d, n), dtype=F64, device=plan.device)
    if not plan.cell_cross:
        return du.t(), 0.0
    dnu = torch.zeros(1, dtype=F64, device=plan.device)
    _lib.call("pf_adj_momentum_cross", plan.handle,
              _lib.ptr(soa(u_cross, n, d, plan.device)), float(nu),
              _lib.ptr(soa(cot_out, n, d, plan.device)), _lib.ptr(du), 1,
              _lib.ptr(dnu), _lib.ptr(plan.workspace), plan.stream)
    return du.t(), float(dnu.item())


def backward_pressure_solve(domain, p_data, p_sol, cot_p, tol=None,
                            maxiter=None, reports=None):
    """Adjoint of the zero-mean pressure solve (S/adjoint.py:94-113):
    project cot_p to zero mean, solve (-P) y = chat with the same operator,
    dP = y (x) p on the pattern, db = -y.  ``p_data`` is the P stencil
    (2d+1, n) (tape.p_data); dP is returned in face form (2d, n): dP[f, i]
    = y_i (p_nb(i,f) - p_i), the on-pattern values folded with the diagonal
    as backward_pressure_matrix consumes them.  Returns (dP, db)."""
    plan = domain.device_plan(cot_p.device)
    n, d = domain.n, domain.dim
    chat = scalar_field(cot_p, n, plan.device)
    chat = chat - chat.mean()
    dkf = torch.zeros((2 * d, n), dtype=F64, device=plan.device)
    if not bool(torch.any(chat != 0)):
        return dkf, torch.zeros(n, dtype=F64, device=plan.device)
    y, rep = cg_solve(plan, -p_data, chat, tol=tol, maxiter=maxiter,
                      zero_mean=True, stage="adjoint_pressure")
    if reports is not None:
        reports.append(rep)
    _lib.call("pf_bwd_pressure_outer", plan.handle, _lib.ptr(y),
              _lib.ptr(scalar_field(p_sol, n, plan.device)), _lib.ptr(dkf),
              0, plan.stream)
    return dkf, -y


def backward_pressure_matrix(domain, a_inv, dP):
    """Chain dP (face form, from backward_pressure_solve) through the
    face-mean pressure assembly back to the diagonal A (S/adjoint.py:
    116-134): returns -a_inv^2 g_ainv, the cotangent of A."""
    from .piso import _cdiag
    plan = domain.device_plan(dP.device)
    n = domain.n
    ainv = scalar_field(a_inv, n, plan.device)
    da = torch.zeros(n, dtype=F64, device=plan.device)
    _lib.call("pf_bwd_pressure_matrix", plan.handle,
              _lib.ptr(_cdiag(1.0 / ainv, n, plan.device)),
              _lib.ptr(dP.contiguous()), _lib.ptr(da), plan.stream)
    return da


def backward_rollout(domain, tapes, cots, path=GradientPath.FULL, tol=None,
                     maxiter=None):
    """Reverse chain over recorded steps (S/adjoint.py:509-539): u is the
    cotangent of the initial velocity; nu, source and bc accumulate."""
    if len(tapes) != len(cots):
        raise ValueError("need one cotangent slot per recorded step")
    n, d = domain.n, domain.dim
    dev = tapes[-1].c_data.device if tapes else None
    total = GradState.zeros(domain, dev)
    src = total.source.t()           # (d, n) storage
    bc_total = [b for b in total.bc]
    cu = torch.zeros((d, n), dtype=F64, device=dev)
    for k in reversed(range(len(tapes))):
        ck = cots[k]
        if ck is not None:
            cu = cu + soa(ck.u, n, d, dev)
            cp = ck.p
        else:
            cp = None
        g = backward_step(domain, tapes[k], GradState(u=cu.t(), p=cp),
                          path=path, tol=tol, maxiter=maxiter)
        total.nu += g.nu
        src += g.source.t()
        for i in range(len(bc_total)):
            bc_total[i] += g.bc[i]
        total.solve_iterations += g.solve_iterations
        cu = soa(g.u, n, d, dev)
    total.u = cu.t()
    return total


# ---------------------------------------------------------------------------
# finite-difference verification harness (S/adjoint.py:546-624)


@dataclass
class GradcheckEntry:
    stage: str
    name: str
    max_rel_err: float
    passed: bool


@dataclass
class GradcheckReport:
    entries: list = field(default_factory=list)
    threshold: float = 1e-4

    @property
    def passed(self):
        return all(e.passed for e in self.entries)

    @property
    def max_rel_err(self):
        return max((e.max_rel_err for e in self.entries), default=0.0)

    def text(self):
        return "\n".join(
            f"stage={e.stage} input={e.name} max_rel_err={e.max_rel_err:.3e} "
            f"pass={1 if e.passed else 0}" for e in self.entries)


def _to_np(x):
    if torch.is_tensor(x):
        return x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def gradcheck(fn, inputs, eps=None, mode="central", threshold=1e-4,
              stage="map"):
    """Central (or forward) finite differences against the analytic
    gradient; relative error floored at 10% of the largest magnitude per
    input (the reference's acceptance metric)."""
    names = list(inputs)
    is_scalar = {k: np.ndim(_to_np(inputs[k])) == 0 for k in names}
    work = {k: np.array(np.atleast_1d(_to_np(inputs[k])), dtype=np.float64)
            for k in names}

    def evaluate():
        args = {k: (float(work[k][0]) if is_scalar[k] else work[k].copy())
                for k in names}
        return float(fn(args)[0])

    loss0, grads = fn(inputs)
    rep = GradcheckReport(threshold=threshold)
    base_eps = float(np.cbrt(np.finfo(np.float64).eps))
    for k in names:
        g_an = np.atleast_1d(_to_np(grads[k])).astype(np.float64)
        flat = work[k].reshape(-1)
        g_fd = np.zeros(flat.size)
        for j in range(flat.size):
            h = eps if eps is not None else base_eps * max(1.0, abs(flat[j]))
            keep = flat[j]
            flat[j] = keep + h
            up = evaluate()
            if mode == "central":
                flat[j] = keep - h
                g_fd[j] = (up - evaluate()) / (2.0 * h)
            else:
                g_fd[j] = (up - loss0) / h
            flat[j] = keep
        g_fd = g_fd.reshape(g_an.shape)
        if not (np.isfinite(g_an).all() and np.isfinite(g_fd).all()):
            rep.entries.append(GradcheckEntry(stage, k, float("inf"), False))
            continue
        scale = max(np.abs(g_an).max(), np.abs(g_fd).max(), 1e-12)
        err = np.abs(g_an - g_fd) / np.maximum(np.abs(g_fd), 0.1 * scale)
        worst = float(err.max()) if err.size else 0.0
        rep.entries.append(GradcheckEntry(stage, k, worst, worst <= threshold))
    return rep



from .piso import _traced  # noqa: E402

backward_step = _traced(backward_step, "backward_step")

__all__ = ["GradientPath", "GradState", "backward_step", "backward_rollout",
           "GradcheckEntry", "GradcheckReport", "gradcheck",
           "backward_correct_velocity", "backward_pressure_solve",
           "backward_pressure_matrix"]
