"""Krylov solvers on device stencils (mirror of S/linalg.py).

``cg_solve`` and ``bicgstab_solve`` keep the reference's signatures and
semantics (relative tolerance, ``maxiter = max(200, 40 round(sqrt n))``,
zero-mean projection, true-residual verification <= 10 tol_abs, retry
unpreconditioned from zero with 2*maxiter, ``SolverError`` carrying a
``SolverReport``).  The operator is a (2d+1, n) stencil on a
:class:`~paper_2505_16992_b200.plan.DevicePlan`; the preconditioner is Jacobi
(``precond="ilu0"``, the reference's default name, selects it; ``None``
runs unpreconditioned).  All iteration happens inside ``libpisob200.so``.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


class SolverError(RuntimeError):
    """A linear solve failed even after the fallback retry
    (S/linalg.py:18-26)."""

    def __init__(self, report):
        self.report = report
        super().__init__(
            f"linear solve '{report.stage}' failed: residual "
            f"{report.residual:.3e} after {report.iterations} iterations"
            + (" (fallback tried)" if report.fallback_used else ""))


@dataclass
class SolverReport:
    converged: bool
    iterations: int
    residual: float
    fallback_used: bool = False
    stage: str = ""


def default_tol(dtype=np.float64):
    """1e-5 for fp32 systems, 1e-8 otherwise (S/linalg.py:125-126)."""
    if dtype in (np.float32, torch.float32) or str(dtype) == "float32":
        return 1e-5
    return 1e-8


def default_maxiter(n):
    return max(200, 40 * int(round(n ** 0.5)))


def _global_n(plan):
    """Cell count of the whole system: a slab plan (one rank's planes plus
    ghosts) takes the global domain's, so every rank -- and the
    single-GPU / reference solve -- gets the same default maxiter (a rank
    stopping early would leave its peers waiting in the cross-rank
    reductions)."""
    g = getattr(plan.domain, "global_domain", None)
    return g.n if g is not None else plan.n


PRECOND_NONE, PRECOND_JACOBI, PRECOND_MG, PRECOND_NEUMANN2 = 0, 1, 2, 3
_DEFAULT_MOM_PRECOND = os.environ.get("PF_MOMENTUM_PRECOND", "neumann2")
# slab plans of more than one rank: Jacobi unless PF_MOMENTUM_PRECOND names
# the polynomial explicitly -- its edge passes and the extra exchanges of
# their stage-1 planes cost more than the halved iteration count saves
# (profiles/r2_s4/slab_overhead_*: C4 as 2 / 8 slabs 37.6 / 51.8 ms per step
# with Jacobi against 39.4 / 54.0 with Neumann-2)
_SLAB_MOM_PRECOND = os.environ.get("PF_MOMENTUM_PRECOND", "jacobi")
# PF_PRESSURE_PRECOND=jacobi: Jacobi-PCG for the pressure even where the
# plan has a spectral / multigrid preconditioner (A/B and debugging)
_DEFAULT_P_PRECOND = os.environ.get("PF_PRESSURE_PRECOND", "auto")


def _precond_flag(precond):
    """None -> unpreconditioned; "jacobi" -> Jacobi; "mg" -> multigrid;
    "ilu0" (the reference's default name) / "auto" -> multigrid where the
    plan supports it for this solve, Jacobi otherwise."""
    if precond is None:
        return PRECOND_NONE
    if precond in ("jacobi",):
        return PRECOND_JACOBI
    if precond in ("mg", "multigrid"):
        return PRECOND_MG
    if precond in ("neumann2", "poly2"):
        return PRECOND_NEUMANN2
    return -1        # auto


def auto_momentum_precond(plan):
    """The momentum BiCGStab preconditioner "ilu0" / "auto" resolves to:
    Neumann-2 on one domain, Jacobi on slab plans of several ranks (the
    library degrades Neumann-2 to Jacobi where its tiled passes do not
    run); PF_MOMENTUM_PRECOND overrides both."""
    multi = getattr(plan.domain, "world", 1) > 1
    pick = _SLAB_MOM_PRECOND if multi else _DEFAULT_MOM_PRECOND
    return PRECOND_NEUMANN2 if pick == "neumann2" else PRECOND_JACOBI


def _report(c, stage):
    return SolverReport(converged=bool(c.converged),
                        iterations=int(c.iterations),
                        residual=float(c.residual),
                        fallback_used=bool(c.fallback_used), stage=stage)


def cg_solve(plan, data, b, x0=None, tol=None, maxiter=None,
             precond="ilu0", zero_mean=False, stage="cg",
             raise_on_fail=True, b_scale=1.0, out=None):
    """Preconditioned CG for the SPD (or zero-mean singular) stencil
    ``data`` (S/linalg.py:258-273).  Solves A x = b_scale * b."""
    n = plan.n
    tol = default_tol() if tol is None else float(tol)
    maxiter = default_maxiter(_global_n(plan)) if maxiter is None \
        else int(maxiter)
    x = torch.empty(n, dtype=torch.float64, device=plan.device) \
        if out is None else out
    if x0 is not None:
        x.copy_(x0)
    pc = _precond_flag(precond)
    if pc == -1:
        # multigrid is built for the zero-mean pressure operator (symmetric
        # face form with zero row sums); everything else gets Jacobi
        pc = PRECOND_MG if (zero_mean and plan.has_mg and
                            _DEFAULT_P_PRECOND != "jacobi") else PRECOND_JACOBI
    mgw = None
    if pc == PRECOND_MG:
        if not plan.mg_prepare(data):
            raise ValueError("multigrid preconditioner unavailable for this "
                             "domain")
        mgw = plan.mg_workspace
    rep = _lib.SolverReportC()
    with _lib.nvtx(stage):
        _lib.call("pf_cg_solve", plan.handle, _lib.ptr(data), _lib.ptr(b),
                  float(b_scale), _lib.ptr(x), int(x0 is not None), tol,
                  maxiter, int(bool(zero_mean)), pc,
                  _lib.ptr(plan.workspace), _lib.ptr(mgw), ctypes.byref(rep),
                  plan.stream)
    report = _report(rep, stage)
    if not report.converged and raise_on_fail:
        raise SolverError(report)
    return x, report


def bicgstab_solve(plan, data, b, x0=None, tol=None, maxiter=None,
                   precond="ilu0", stage="bicgstab", raise_on_fail=True,
                   transpose=False, stages=None, out=None):
    """Right-preconditioned BiCGStab (S/linalg.py:276-281) on k right-hand
    sides at once: ``b`` is (k, n) (or (n,)), every row an independent
    solve sharing the matrix.  Returns (x, [SolverReport] * k)."""
    n = plan.n
    squeeze = b.dim() == 1
    b2 = b.reshape(-1, n)
    k = b2.shape[0]
    tol = default_tol() if tol is None else float(tol)
    maxiter = default_maxiter(_global_n(plan)) if maxiter is None \
        else int(maxiter)
    x = torch.empty((k, n), dtype=torch.float64, device=plan.device) \
        if out is None else out.reshape(k, n)
    if x0 is not None:
        x.copy_(x0.reshape(k, n))
    reps = (_lib.SolverReportC * k)()
    pc = _precond_flag(precond)
    # auto / "ilu0": the fused two-sweep Jacobi polynomial (Neumann-2) on
    # tiled boxes (the library degrades it to Jacobi elsewhere): C4
    # lock-step iterations 15 -> 8 per step; same-box A/B 31.0 ms vs 32.0
    # ms with Jacobi (profiles/r2_nm_light.txt).  PF_MOMENTUM_PRECOND=jacobi
    # selects Jacobi
    if pc == -1:
        pc = auto_momentum_precond(plan)
    elif pc == PRECOND_MG:
        pc = PRECOND_JACOBI
    with _lib.nvtx(stages[0] if stages else stage):
        _lib.call("pf_bicgstab_solve", plan.handle, _lib.ptr(data),
                  int(bool(transpose)), k, _lib.ptr(b2), _lib.ptr(x),
                  int(x0 is not None), tol, maxiter, pc,
                  _lib.ptr(plan.workspace), reps, plan.stream)
    if stages is None:
        stages = [stage] * k
    reports = [_report(reps[q], stages[q]) for q in range(k)]
    if raise_on_fail:
        for r in reports:
            if not r.converged:
                raise SolverError(r)
    return (x[0] if squeeze else x), reports


def stencil_matvec(plan, data, x, transpose=False, out=None):
    """y = A x (or A^t x) for a (2d+1, n) stencil; x is (n,) or (k, n)."""
    n = plan.n
    x2 = x.reshape(-1, n)
    y = torch.empty_like(x2) if out is None else out.reshape(x2.shape)
    _lib.call("pf_stencil_matvec", plan.handle, _lib.ptr(data),
              int(bool(transpose)), x2.shape[0], _lib.ptr(x2), _lib.ptr(y),
              plan.stream)
    return y.reshape(x.shape)


def stencil_to_csr(domain, stencil):
    """(2d+1, n) stencil -> scipy CSR on the cell-adjacency pattern (host;
    for comparisons against the reference's CSR ``data`` arrays)."""
    import scipy.sparse as sp
    st = stencil.detach().cpu().numpy() if torch.is_tensor(stencil) \
        else np.asarray(stencil)
    d, n = domain.dim, domain.n
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    vals = [st[0]]
    for f in range(2 * d):
        a, s = divmod(f, 2)
        nb = domain.nbr[a, s]
        ok = nb >= 0
        rows.append(np.nonzero(ok)[0])
        cols.append(nb[ok])
        vals.append(st[1 + f][ok])
    return sp.csr_matrix((np.concatenate(vals),
                          (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n))
