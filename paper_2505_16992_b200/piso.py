"""The PISO time step on device (mirror of S/piso.py).

``piso_step(domain, state, cfg, workspace=None, tape=None)`` keeps the
reference's signature, defaults, error behaviour and stage labels
(S/piso.py:561-654); every arithmetic stage is a kernel of
``libpisob200.so``:

=====================  ==========================================  =================
stage                  reference                                   kernel entry
=====================  ==========================================  =================
outflow preprocess     advective_outflow_update  S/piso.py:467     pf_advective_outflow_update
momentum matrix        assemble_momentum         S/piso.py:293     pf_assemble_momentum
predictor rhs          momentum_rhs              S/piso.py:356     pf_momentum_rhs
predictor solves       bicgstab_solve x d        S/piso.py:583     pf_bicgstab_solve (d batched)
pressure matrix        assemble_pressure         S/piso.py:395     pf_assemble_pressure
h stage                C u - A u, A^-1(rhs-Hu)   S/piso.py:608     pf_h_stage
divergence rhs         divergence_rhs            S/piso.py:415     pf_divergence_rhs
pressure solve         cg_solve zero-mean        S/piso.py:619     pf_cg_solve
projection             correct_velocity          S/piso.py:452     pf_correct_velocity
diagnostic             divergence max            S/piso.py:635     pf_divergence_max
=====================  ==========================================  =================

Fields are torch float64 tensors on the plan's CUDA device.  Vector fields
are stored structure-of-arrays (d, n) and exposed as the reference's (n, d)
through transposed views, so ``state.u[i, c]`` reads what the reference
would.  Matrices are (2d+1, n) stencils (row 0 the diagonal, row 1+f the
face-f neighbour coupling) instead of CSR ``data`` arrays; the tape holds
K = -P (the operator the pressure CG runs on) and exposes ``p_data = -K``.

Non-orthogonal grids (alpha with off-diagonal entries, e.g. the distorted
Poiseuille duct) run the lagged cross fluxes of S/piso.py:322-353,431-449
and the ``nonortho_correctors`` loops on the device (csrc/cross.cu).

Slab domains (slab.SlabDomain, one per GPU) run this same code: the library
exchanges ghost planes and reduces across the ranks inside its entry points.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .linalg import SolverError, bicgstab_solve, cg_solve

F64 = torch.float64


# ---------------------------------------------------------------------------
# layout helpers


def soa(x, n, d, device):
    """(n, d) array/tensor -> contiguous (d, n) float64 tensor on device
    (free when x is already a transposed view of such a tensor)."""
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64))
    x = x.to(device=device, dtype=F64)
    if x.shape != (n, d):
        raise ValueError(f"expected an ({n}, {d}) field, got {tuple(x.shape)}")
    t = x.t()
    return t if t.is_contiguous() else t.contiguous()


def scalar_field(x, n, device):
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64))
    x = x.to(device=device, dtype=F64).reshape(n)
    return x if x.is_contiguous() else x.contiguous()


def bc_soa(plan, bc, d):
    """Per-face list of (m_f, d) boundary velocities -> one (d, m) tensor."""
    if plan.m == 0:
        return None
    parts = [(b if torch.is_tensor(b) else torch.as_tensor(
        np.asarray(b, dtype=np.float64))).to(plan.device, F64).reshape(-1, d)
        for b in bc]
    return torch.cat(parts, dim=0).t().contiguous()


def bc_views(plan, bc_dm):
    """(d, m) tensor -> list of (m_f, d) views in domain.bfaces order."""
    if bc_dm is None:
        return []
    off = plan.face_offsets
    return [bc_dm[:, off[k]:off[k + 1]].t() for k in range(len(off) - 1)]


# ---------------------------------------------------------------------------
# state, config, tape


@dataclass
class FlowState:
    u: torch.Tensor          # (n, d) Cartesian velocity
    p: torch.Tensor          # (n,) pressure of the last corrector
    bc: list                 # per boundary face, (m, d) face velocities
    t: float = 0.0
    step: int = 0

    def copy(self):
        def cp(x):
            return x.t().clone().t() if x.dim() == 2 else x.clone()
        return FlowState(cp(self.u), self.p.clone(), [cp(b) for b in self.bc],
                         self.t, self.step)


@dataclass
class StepConfig:
    dt: float
    nu: float
    n_correctors: int = 2
    nonortho_correctors: int = 0
    source: object = None    # None, (d,) or (n, d)
    tol: float = None
    maxiter: int = None


@dataclass
class StepDiagnostics:
    dt: float = 0.0
    advout_scale: float = 1.0
    momentum_iterations: int = 0
    pressure_iterations: int = 0
    div_contract: float = 0.0
    # a float, or the device scalar pf_divergence_max_dev wrote (read on
    # first access, so the step itself never waits for it)
    _div_wide_max: object = 0.0
    reports: list = field(default_factory=list)

    @property
    def div_wide_max(self) -> float:
        v = self._div_wide_max
        if torch.is_tensor(v):
            v = self._div_wide_max = float(v.item())
        return v

    @div_wide_max.setter
    def div_wide_max(self, value):
        self._div_wide_max = value


@dataclass
class CorrectorTape:
    u_hin: torch.Tensor      # (n, d) velocity whose H u enters h
    h: torch.Tensor          # (n, d)
    p_iters: list            # pressure iterates, last one applied


@dataclass
class StepTape:
    dt: float = 0.0
    nu: float = 0.0
    source: torch.Tensor = None      # (n, d)
    u_n: torch.Tensor = None         # (n, d)
    bc: list = None
    c_data: torch.Tensor = None      # (2d+1, n) momentum stencil
    a_diag: torch.Tensor = None      # (n,) view of c_data[0]
    rhs_final: torch.Tensor = None   # (n, d)
    mom_inputs: list = None
    mom_iters: list = None
    k_data: torch.Tensor = None      # (2d+1, n) stencil of K = -P
    correctors: list = None
    u_out: torch.Tensor = None

    @property
    def p_data(self):
        return None if self.k_data is None else -self.k_data


class PisoWorkspace:
    """Per-domain warm starts (S/piso.py:90-103); device tensors."""

    def __init__(self, domain, warm_starts=True):
        self.domain = domain
        self.warm_starts = warm_starts
        self._warm = {}

    def warm(self, key):
        return self._warm.get(key) if self.warm_starts else None

    def store(self, key, x):
        if self.warm_starts:
            self._warm[key] = x.clone()


def _default_device(device):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda", torch.cuda.current_device()) \
        if torch.cuda.is_available() else torch.device("cuda")


def make_state(domain, u0=None, p0=None, t=0.0, device=None):
    """Initial state (S/piso.py:106-116); outflow faces are seeded from the
    adjacent cells."""
    dev = _default_device(device)
    _lib.require_cuda(dev)
    n, d = domain.n, domain.dim
    if u0 is None:
        u = torch.zeros((d, n), dtype=F64, device=dev)
    else:
        u = soa(u0, n, d, dev).clone()
    p = torch.zeros(n, dtype=F64, device=dev) if p0 is None else \
        scalar_field(p0, n, dev).clone()
    u_host = None
    bc = []
    for f in domain.bfaces:
        vals = f.initial_values(d)
        if vals is None:
            if u_host is None:
                u_host = u.t().cpu().numpy()
            vals = u_host[f.cells].copy()
        bc.append(vals)
    plan = domain.device_plan(dev)
    return FlowState(u.t(), p, bc_views(plan, bc_soa(plan, bc, d)), t=t,
                     step=0)


# ---------------------------------------------------------------------------
# building blocks (kernel wrappers; inputs/outputs in the reference layout)


def _plan_of(domain, x):
    return domain.device_plan(x.device)


def contravariant_flux(domain, u):
    plan = _plan_of(domain, u)
    n, d = domain.n, domain.dim
    out = torch.empty((d, n), dtype=F64, device=plan.device)
    _lib.call("pf_contravariant_flux", plan.handle,
              _lib.ptr(soa(u, n, d, plan.device)), _lib.ptr(out), plan.stream)
    return out.t()


def assemble_momentum(domain, u_n, nu, dt):
    """Momentum stencil (2d+1, n) (S/piso.py:293-319)."""
    plan = _plan_of(domain, u_n)
    n, d = domain.n, domain.dim
    c = torch.empty((2 * d + 1, n), dtype=F64, device=plan.device)
    flux = torch.empty((d, n), dtype=F64, device=plan.device)
    _lib.call("pf_assemble_momentum", plan.handle,
              _lib.ptr(soa(u_n, n, d, plan.device)), float(nu), float(dt),
              _lib.ptr(flux), _lib.ptr(c), plan.stream)
    return c


def assemble_pressure(domain, a_inv):
    """P stencil (2d+1, n) from A^-1 (S/piso.py:395-412)."""
    plan = _plan_of(domain, a_inv)
    n, d = domain.n, domain.dim
    k = torch.empty((2 * d + 1, n), dtype=F64, device=plan.device)
    _lib.call("pf_assemble_pressure", plan.handle,
              _lib.ptr(scalar_field(a_inv, n, plan.device)), 1, _lib.ptr(k),
              plan.stream)
    return -k


def momentum_rhs(domain, u_n, bc, nu, dt, source, u_cross=None):
    """Predictor right-hand side (S/piso.py:356-372), orthogonal grids."""
    plan = _plan_of(domain, u_n)
    n, d = domain.n, domain.dim
    src, uniform = _resolve_source(domain, source, plan.device)
    out = torch.empty((d, n), dtype=F64, device=plan.device)
    bcd = bc_soa(plan, bc, d)
    _lib.call("pf_momentum_rhs", plan.handle,
              _lib.ptr(soa(u_n, n, d, plan.device)), _lib.ptr(bcd),
              _lib.ptr(src), uniform, float(nu), float(dt), _lib.ptr(out),
              plan.stream)
    return out.t()


def divergence_rhs(domain, h, bc):
    """xi-space flux divergence with boundary fluxes (S/piso.py:415-428)."""
    plan = _plan_of(domain, h)
    n, d = domain.n, domain.dim
    b = torch.empty(n, dtype=F64, device=plan.device)
    flux = torch.empty((d, n), dtype=F64, device=plan.device)
    _lib.call("pf_divergence_rhs", plan.handle,
              _lib.ptr(soa(h, n, d, plan.device)),
              _lib.ptr(bc_soa(plan, bc, d)), _lib.ptr(flux), _lib.ptr(b),
              plan.stream)
    return b


def correct_velocity(domain, h, p, a_inv):
    """u = h - A^-1 T^t grad(p) with mirror ghosts (S/piso.py:452-455)."""
    plan = _plan_of(domain, h)
    n, d = domain.n, domain.dim
    # the kernel reads A from the stencil's diagonal row
    cdiag = (1.0 / scalar_field(a_inv, n, plan.device)).reshape(1, n)
    out = torch.empty((d, n), dtype=F64, device=plan.device)
    _lib.call("pf_correct_velocity", plan.handle,
              _lib.ptr(soa(h, n, d, plan.device)),
              _lib.ptr(scalar_field(p, n, plan.device)),
              _lib.ptr(cdiag.contiguous()), _lib.ptr(out), plan.stream)
    return out.t()


# ---------------------------------------------------------------------------
# standalone building blocks of the reference's stage API (S/piso.py:128-264,
# 322-342, 431-449); the step uses their fused forms

WIDE_GRAD_VARIANTS = {"mirror": 0, "onesided": 1, "face": 2}


def _variant(variant):
    try:
        return WIDE_GRAD_VARIANTS[variant]
    except KeyError:
        raise ValueError(variant) from None


def boundary_flux(face, values):
    """U^a at a boundary face from prescribed face velocities (m, d)
    (S/piso.py:128-131)."""
    dev = values.device
    jac = torch.as_tensor(face.face_jac, dtype=F64, device=dev)
    t = torch.as_tensor(np.ascontiguousarray(face.face_t[:, face.axis, :]),
                        dtype=F64, device=dev)
    return jac * (t * values).sum(dim=1)


def face_grad(arr, axis):
    """Derivative along one axis of a face-value grid: central inside, full
    one-sided at the ends (S/piso.py:134-145)."""
    a = arr.movedim(axis, 0)
    out = torch.empty_like(a)
    if a.shape[0] == 1:
        out.zero_()
    else:
        out[1:-1] = 0.5 * (a[2:] - a[:-2])
        out[0] = a[1] - a[0]
        out[-1] = a[-1] - a[-2]
    return out.movedim(0, axis)


def face_grad_adjoint(cot, axis):
    """Adjoint of :func:`face_grad` (S/piso.py:148-159)."""
    c = cot.movedim(axis, 0)
    out = torch.zeros_like(c)
    if c.shape[0] > 1:
        out[2:] += 0.5 * c[1:-1]
        out[:-2] -= 0.5 * c[1:-1]
        out[1] += c[0]
        out[0] -= c[0]
        out[-1] += c[-1]
        out[-2] -= c[-1]
    return out.movedim(0, axis)


def wide_grad(domain, phi, variant, bc_cells=None):
    """Wide central differences of a per-cell field along every grid axis
    (S/piso.py:172-209): (n,) -> (n, d); (n, k) -> (n, d, k).  variant
    "mirror" | "onesided" | "face" (``bc_cells``: {(axis, side): (n,)}
    prescribed face values).  Kernel: pf_wide_grad."""
    plan = _plan_of(domain, phi)
    n, d = domain.n, domain.dim
    v = _variant(variant)
    bcc = None
    if v == 2:
        if bc_cells is None:
            raise ValueError("the face variant needs bc_cells")
        bcc = torch.stack([torch.as_tensor(bc_cells[(a, s_)], dtype=F64,
                                           device=plan.device).reshape(n)
                           for a in range(d) for s_ in (0, 1)]).contiguous()
    cols = [phi] if phi.dim() == 1 else [phi[:, k] for k in
                                         range(phi.shape[1])]
    outs = []
    for col in cols:
        out = torch.empty((d, n), dtype=F64, device=plan.device)
        _lib.call("pf_wide_grad", plan.handle,
                  _lib.ptr(scalar_field(col, n, plan.device)), v,
                  _lib.ptr(bcc), _lib.ptr(out), plan.stream)
        outs.append(out.t())
    return outs[0] if phi.dim() == 1 else torch.stack(outs, dim=2)


def wide_grad_adjoint(domain, cot, variant, phi_ndim=1):
    """Adjoint of :func:`wide_grad` w.r.t. phi (S/piso.py:218-258): cot
    (n, d[, k]) -> (n[, k]); the face variant also returns {(axis, side):
    (n,)} cotangents of the prescribed face values.  Kernel:
    pf_wide_grad_adjoint."""
    plan = _plan_of(domain, cot)
    n, d = domain.n, domain.dim
    v = _variant(variant)
    cols = [cot] if cot.dim() == 2 else [cot[:, :, k] for k in
                                         range(cot.shape[2])]
    outs, bcs = [], []
    for col in cols:
        out = torch.empty(n, dtype=F64, device=plan.device)
        bc = torch.empty((2 * d, n), dtype=F64, device=plan.device) \
            if v == 2 else None
        _lib.call("pf_wide_grad_adjoint", plan.handle,
                  _lib.ptr(soa(col, n, d, plan.device)), v, _lib.ptr(out),
                  _lib.ptr(bc), plan.stream)
        outs.append(out)
        bcs.append(bc)
    res = outs[0] if cot.dim() == 2 else torch.stack(outs, dim=1)
    if v != 2:
        return res
    bcr = bcs[0] if cot.dim() == 2 else torch.stack(bcs, dim=2)
    return res, {(a, s_): bcr[2 * a + s_] for a in range(d) for s_ in (0, 1)}


def _cdiag(a_diag, n, device):
    """A stencil carrying only the diagonal row (kernels read A from row 0)."""
    return scalar_field(a_diag, n, device).reshape(1, n).contiguous()


def momentum_cross_rhs(domain, u, nu):
    """Lagged non-orthogonal viscous fluxes divided by J (S/piso.py:322-342),
    (n, d); zero on orthogonal grids.  Kernel: pf_momentum_cross_rhs."""
    plan = _plan_of(domain, u)
    n, d = domain.n, domain.dim
    out = torch.zeros((d, n), dtype=F64, device=plan.device)
    if plan.cell_cross:
        _lib.call("pf_momentum_cross_rhs", plan.handle,
                  _lib.ptr(soa(u, n, d, plan.device)), float(nu),
                  _lib.ptr(out), _lib.ptr(plan.workspace), plan.stream)
    return out.t()


def pressure_cross_rhs(domain, a_inv, p):
    """Lagged non-orthogonal pressure fluxes (S/piso.py:431-449), (n,);
    zero on orthogonal grids.  Kernel: pf_pressure_cross_rhs."""
    plan = _plan_of(domain, p)
    n = domain.n
    if not plan.cell_cross:
        return torch.zeros(n, dtype=F64, device=plan.device)
    c = _cdiag(1.0 / scalar_field(a_inv, n, plan.device), n, plan.device)
    zero = torch.zeros(n, dtype=F64, device=plan.device)
    out = torch.empty(n, dtype=F64, device=plan.device)
    _lib.call("pf_pressure_cross_rhs", plan.handle, _lib.ptr(c),
              _lib.ptr(scalar_field(p, n, plan.device)), _lib.ptr(zero),
              _lib.ptr(out), _lib.ptr(plan.workspace), plan.stream)
    return -out


def divergence(domain, u, bc):
    """Per-cell physical divergence (S/piso.py:458-460)."""
    return divergence_rhs(domain, u, bc) / domain.device_plan(u.device).jac


def advective_outflow_update(domain, state, dt):
    """Outflow relaxation + mass rebalance (S/piso.py:467-509); returns
    (bc list, scale) without modifying ``state``."""
    plan = domain.device_plan(state.u.device)
    d = domain.dim
    bcd = bc_soa(plan, state.bc, d)
    if not plan.has_outflow:
        return bc_views(plan, bcd), 1.0
    scale = _lib.c_dbl()
    _lib.call("pf_advective_outflow_update", plan.handle,
              _lib.ptr(soa(state.u, domain.n, d, plan.device)), _lib.ptr(bcd),
              float(dt), _lib.ptr(plan.workspace), _lib.ctypes.byref(scale),
              plan.stream)
    return bc_views(plan, bcd), float(scale.value)


def _resolve_source(domain, source, device):
    """(tensor, uniform flag): a (d,) vector stays a vector, an (n, d) field
    becomes (d, n) SoA (S/piso.py:549-558 semantics)."""
    n, d = domain.n, domain.dim
    if source is None:
        return torch.zeros(d, dtype=F64, device=device), 1
    src = source if torch.is_tensor(source) else torch.as_tensor(
        np.asarray(source, dtype=np.float64))
    src = src.to(device=device, dtype=F64)
    if tuple(src.shape) == (d,):
        return src.contiguous(), 1
    if tuple(src.shape) == (n, d):
        return soa(src, n, d, device), 0
    raise ValueError(f"source shape {tuple(src.shape)} does not fit "
                     f"({n}, {d})")


# ---------------------------------------------------------------------------
# the step


def piso_step(domain, state, cfg, workspace=None, tape=None):
    """Advance one time step; optionally record a tape for reverse mode
    (S/piso.py:561-654)."""
    ws = workspace or PisoWorkspace(domain, warm_starts=False)
    dt, nu = float(cfg.dt), float(cfg.nu)
    if dt <= 0 or nu <= 0:
        raise ValueError("dt and nu must be positive")
    if not torch.is_tensor(state.u):
        # a reference-style state of NumPy arrays: move it to the device
        dev = _default_device(None)
        plan0 = domain.device_plan(dev)
        state = FlowState(soa(state.u, domain.n, domain.dim, dev).t(),
                          scalar_field(state.p, domain.n, dev),
                          bc_views(plan0, bc_soa(plan0, state.bc,
                                                 domain.dim)),
                          state.t, state.step)
    dev = state.u.device
    _lib.require_cuda(dev)
    plan = domain.device_plan(dev)
    n, d = domain.n, domain.dim
    hstream = plan.stream
    diag = StepDiagnostics(dt=dt)
    src, uniform = _resolve_source(domain, cfg.source, dev)

    # boundary preprocessing (not differentiated)
    u_n = soa(state.u, n, d, dev)
    bc = bc_soa(plan, state.bc, d)
    if plan.has_outflow:
        scale = _lib.c_dbl()
        _lib.call("pf_advective_outflow_update", plan.handle, _lib.ptr(u_n),
                  _lib.ptr(bc), dt, _lib.ptr(plan.workspace),
                  _lib.ctypes.byref(scale), hstream)
        diag.advout_scale = float(scale.value)

    flux = torch.empty((d, n), dtype=F64, device=dev)
    c_data = torch.empty((2 * d + 1, n), dtype=F64, device=dev)
    _lib.call("pf_assemble_momentum", plan.handle, _lib.ptr(u_n), nu, dt,
              _lib.ptr(flux), _lib.ptr(c_data), hstream)

    n_outer = 1 + int(cfg.nonortho_correctors)
    mom_inputs, mom_iters = [], []
    u_prev = u_n
    u_star = None
    stages = [f"momentum[{c}]" for c in range(d)]
    for _ in range(n_outer):
        # rhs = u_n/dt + S + boundary terms (+ the lagged cross flux of the
        # previous outer iterate on non-orthogonal grids, S/piso.py:582)
        rhs = torch.empty((d, n), dtype=F64, device=dev)
        _lib.call("pf_momentum_rhs", plan.handle, _lib.ptr(u_n),
                  _lib.ptr(bc), _lib.ptr(src), uniform, nu, dt,
                  _lib.ptr(rhs), hstream)
        if plan.cell_cross:
            _lib.call("pf_momentum_cross_rhs", plan.handle, _lib.ptr(u_prev),
                      nu, _lib.ptr(rhs), _lib.ptr(plan.workspace), hstream)
        u_star, reps = bicgstab_solve(plan, c_data, rhs,
                                      x0=ws.warm(("mom",)), tol=cfg.tol,
                                      maxiter=cfg.maxiter, stages=stages)
        for r in reps:
            diag.momentum_iterations += r.iterations
            diag.reports.append(r)
        mom_inputs.append(u_prev.t())
        mom_iters.append(u_star.t())
        u_prev = u_star
    ws.store(("mom",), u_star)

    k_data = torch.empty((2 * d + 1, n), dtype=F64, device=dev)
    _lib.call("pf_assemble_pressure", plan.handle, _lib.ptr(c_data), 0,
              _lib.ptr(k_data), hstream)

    correctors = []
    u_cur = u_star
    p = scalar_field(state.p, n, dev)
    last_resid = 0.0
    b0 = torch.empty(n, dtype=F64, device=dev)
    for m in range(cfg.n_correctors):
        h = torch.empty((d, n), dtype=F64, device=dev)
        _lib.call("pf_h_stage", plan.handle, _lib.ptr(c_data),
                  _lib.ptr(u_cur), _lib.ptr(rhs), _lib.ptr(h), hstream)
        _lib.call("pf_divergence_rhs", plan.handle, _lib.ptr(h),
                  _lib.ptr(bc), _lib.ptr(flux), _lib.ptr(b0), hstream)
        p_iters = []
        for it in range(n_outer):
            b = b0
            if plan.cell_cross and it > 0:
                # b = b0 - lagged pressure cross flux (S/piso.py:617)
                b = torch.empty(n, dtype=F64, device=dev)
                _lib.call("pf_pressure_cross_rhs", plan.handle,
                          _lib.ptr(c_data), _lib.ptr(p_iters[-1]),
                          _lib.ptr(b0), _lib.ptr(b), _lib.ptr(plan.workspace),
                          hstream)
            p_sol, rep = cg_solve(plan, k_data, b, x0=ws.warm(("prs",)),
                                  tol=cfg.tol, maxiter=cfg.maxiter,
                                  zero_mean=True, b_scale=-1.0,
                                  stage=f"pressure[c{m}i{it}]")
            diag.pressure_iterations += rep.iterations
            diag.reports.append(rep)
            p_iters.append(p_sol)
            last_resid = rep.residual
        p = p_iters[-1]
        ws.store(("prs",), p)
        u_new = torch.empty((d, n), dtype=F64, device=dev)
        _lib.call("pf_correct_velocity", plan.handle, _lib.ptr(h),
                  _lib.ptr(p), _lib.ptr(c_data), _lib.ptr(u_new), hstream)
        correctors.append(CorrectorTape(u_hin=u_cur.t(), h=h.t(),
                                        p_iters=p_iters))
        u_cur = u_new

    diag.div_contract = last_resid
    dmax = torch.empty((), dtype=F64, device=dev)
    _lib.call("pf_divergence_max_dev", plan.handle, _lib.ptr(u_cur),
              _lib.ptr(bc), _lib.ptr(flux), _lib.ptr(plan.workspace),
              _lib.ptr(dmax), hstream)
    diag.div_wide_max = dmax

    bc_list = bc_views(plan, bc)
    if tape is not None:
        tape.dt, tape.nu = dt, nu
        tape.source = (src.reshape(1, d).expand(n, d) if uniform
                       else src.t())
        # the reference copies u_n into the tape (S/piso.py:640).  Here u_n
        # may alias the caller's input storage; the adjoint reads it only
        # through the non-orthogonal cross terms (mom_inputs[0]), so it is
        # copied exactly then.  On orthogonal grids the input velocity is
        # not read by backward_step and may be refilled at once.
        if plan.cell_cross and u_n.data_ptr() == state.u.data_ptr():
            u_n = u_n.clone()
            mom_inputs[0] = u_n.t()
        tape.u_n = u_n.t()
        tape.bc = bc_list
        tape.c_data = c_data
        tape.a_diag = c_data[0]
        tape.rhs_final = rhs.t()
        tape.mom_inputs = mom_inputs
        tape.mom_iters = mom_iters
        tape.k_data = k_data
        tape.correctors = correctors
        tape.u_out = u_cur.t()
        tape._bc_dm = bc

    new_state = FlowState(u=u_cur.t(), p=p.clone(), bc=bc_list,
                          t=state.t + dt, step=state.step + 1)
    return new_state, diag



def _traced(fn, name):
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with _lib.nvtx(name):
            return fn(*args, **kwargs)
    return wrapper


piso_step = _traced(piso_step, "piso_step")

__all__ = ["FlowState", "StepConfig", "StepDiagnostics", "CorrectorTape",
           "StepTape", "PisoWorkspace", "make_state", "contravariant_flux",
           "assemble_momentum", "assemble_pressure", "momentum_rhs",
           "divergence_rhs", "correct_velocity", "divergence",
           "advective_outflow_update", "piso_step", "SolverError",
           "boundary_flux", "face_grad", "face_grad_adjoint", "wide_grad",
           "wide_grad_adjoint", "momentum_cross_rhs", "pressure_cross_rhs",
           "reichardt_init", "wall_forcing_source", "adaptive_dt"]


def __getattr__(name):
    # the channel drivers live in channel.py (S/piso.py:512-546, 668-714)
    if name in ("reichardt_init", "reichardt_profile", "wall_forcing_source",
                "adaptive_dt"):
        from . import channel
        return getattr(channel, name)
    raise AttributeError(name)
