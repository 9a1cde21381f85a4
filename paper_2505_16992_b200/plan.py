"""Device-resident plan: the Domain's static arrays in HBM + the C-ABI handle.

Layout in HBM (all fp64 unless noted, SoA so every warp access is
coalesced):

* ``jac`` (n), ``tmat`` (d*d, n) with row ``a*d + j`` = T[:, a, j],
  ``alpha_diag`` (d, n);
* boundary entries in ``domain.bfaces`` order: ``bcell`` int32 (m),
  ``bface`` int32 (m) = face | kind << 4, ``bjac`` (m), ``bt`` (d, m) = the
  face-normal row T_f[a, :], ``balpha`` (m) = alpha_f[a, a];
* gather topology only: ``nbr`` int32 (2d, n), packed neighbour / axis /
  flip / boundary-entry words (see include/pisob200.h).

Solver and reduction scratch (``workspace``) is one zero-initialised byte
tensor sized by ``pf_workspace_bytes``; it is reused by every call on the
plan's stream.
"""

import ctypes

import numpy as np
import torch

from . import _lib


def _spectral_allowed(domain, box, sep):
    """The spectral pressure preconditioner needs a single box whose
    non-line axes (all but the first in 2D, X and Z in 3D) are periodic and
    uniformly spaced; the C library checks the topology (power-of-two
    periodic X / Z), the spacing is asserted here."""
    if box is None or sep is None:
        return False
    shape, periodic = box
    axes = [1] if domain.dim == 2 else [0, 2]
    for a in axes:
        h = np.asarray(sep[a], dtype=np.float64)
        if not periodic[a] or np.ptp(h) > 1e-12 * np.abs(h).max():
            return False
    return True


class DevicePlan:
    """``geom_precond``: "auto" (spectral where the box allows it, else
    multigrid), "multigrid" or "spectral" (falls back to multigrid when the
    box does not allow it)."""

    def __init__(self, domain, device, geom_precond="auto"):
        _lib.require_cuda(device)
        self.domain = domain
        self.device = device
        self.n = n = domain.n
        self.dim = d = domain.dim
        f64 = dict(dtype=torch.float64, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        box = domain.box_layout()
        sep = domain.separable_metrics()

        # --- metrics -------------------------------------------------------
        if box is not None and sep is not None:
            shape = box[0]
            dx = []
            for a in range(d):
                sh = [1] * d
                sh[a] = shape[a]
                dx.append(torch.as_tensor(sep[a], **f64).reshape(sh)
                          .expand(*shape).reshape(-1))
            jac = dx[0].clone()
            for a in range(1, d):
                jac = jac * dx[a]
            tmat = torch.zeros((d * d, n), **f64)
            alpha = torch.empty((d, n), **f64)
            for a in range(d):
                t = 1.0 / dx[a]
                tmat[a * d + a] = t
                alpha[a] = jac * (t * t)
            self.jac, self.tmat, self.alpha_diag = jac, tmat, alpha
            # the 1-D widths the kernels form the same values from
            self.sep_dx = [torch.as_tensor(sep[a], **f64).contiguous()
                           for a in range(d)]
            self.sep_inv = [1.0 / w for w in self.sep_dx]
        else:
            self.jac = torch.as_tensor(domain.jac, **f64).contiguous()
            tm = np.ascontiguousarray(
                domain.tmat.reshape(n, d * d).T)
            self.tmat = torch.as_tensor(tm, **f64)
            al = np.ascontiguousarray(
                domain.alpha[:, np.arange(d), np.arange(d)].T)
            self.alpha_diag = torch.as_tensor(al, **f64)
            self.sep_dx = self.sep_inv = None

        # --- boundary entries ------------------------------------------------
        faces = domain.bfaces
        self.m = m = sum(f.m for f in faces)
        self.face_offsets = domain.bface_offsets
        if m:
            bcell = np.concatenate([f.cells for f in faces]).astype(np.int32)
            kinds = [(_lib.PF_BKIND_DIRICHLET if f.kind == "dirichlet"
                      else _lib.PF_BKIND_OUTFLOW) for f in faces]
            bface = np.concatenate([
                np.full(f.m, (2 * f.axis + f.side) | (k << 4), np.int32)
                for f, k in zip(faces, kinds)])
            bjac = np.concatenate([f.face_jac for f in faces])
            bt = np.concatenate([f.face_t[:, f.axis, :] for f in faces]).T
            balpha = np.concatenate([f.face_alpha[:, f.axis, f.axis]
                                     for f in faces])
            self.bcell = torch.as_tensor(bcell, **i32)
            self.bface = torch.as_tensor(bface, **i32)
            self.bjac = torch.as_tensor(bjac, **f64)
            self.bt = torch.as_tensor(np.ascontiguousarray(bt), **f64)
            self.balpha = torch.as_tensor(balpha, **f64)
        else:
            self.bcell = self.bface = self.bjac = self.bt = self.balpha = None
        self.has_outflow = any(f.kind == "advective_outflow" for f in faces)

        # --- non-orthogonal metric terms ---------------------------------------
        self.cell_cross = domain.cell_cross_terms()
        face_active = [domain.face_cross_active(f) for f in faces]
        self.nonortho = self.cell_cross or any(face_active)
        self.alpha_full = self.balpha_row = self.bfid = self.finfo = None
        if self.nonortho:
            af = np.ascontiguousarray(domain.alpha.reshape(n, d * d).T)
            self.alpha_full = torch.as_tensor(af, **f64)
            if m:
                row = np.concatenate([f.face_alpha[:, f.axis, :]
                                      for f in faces]).T
                self.balpha_row = torch.as_tensor(np.ascontiguousarray(row),
                                                  **f64)
                self.bfid = torch.as_tensor(np.concatenate(
                    [np.full(f.m, k, np.int32) for k, f in enumerate(faces)]),
                    **i32)
                info = np.zeros((len(faces), 8), np.int32)
                for k, (f, off) in enumerate(zip(faces, self.face_offsets)):
                    dims = list(f.area_shape) + [1, 1]
                    info[k] = [off, f.m, dims[0], dims[1], int(face_active[k]),
                               f.axis, f.side, 0]
                self.finfo = torch.as_tensor(info.reshape(-1), **i32)

        # --- topology ----------------------------------------------------------
        desc = _lib.PlanDesc()
        desc.dim = d
        desc.n = n
        if box is not None:
            shape, periodic = box
            desc.topo = _lib.PF_TOPO_BOX
            for a in range(d):
                desc.box_shape[a] = shape[a]
                desc.box_periodic[a] = int(periodic[a])
            offs = [-1] * 6
            for f, off in zip(faces, self.face_offsets):
                offs[2 * f.axis + f.side] = off
            for k in range(6):
                desc.box_face_offset[k] = offs[k]
            self.nbr = None
            self.topo = "box"
        else:
            desc.topo = _lib.PF_TOPO_GATHER
            self.nbr = torch.as_tensor(self._packed_table(), **i32)
            desc.nbr = self.nbr.data_ptr()
            self.topo = "gather"
        desc.jac = self.jac.data_ptr()
        self.ijac = 1.0 / self.jac
        desc.ijac = self.ijac.data_ptr()
        desc.tmat = self.tmat.data_ptr()
        desc.alpha_diag = self.alpha_diag.data_ptr()
        desc.m = m
        if m:
            desc.bcell = self.bcell.data_ptr()
            desc.bface = self.bface.data_ptr()
            desc.bjac = self.bjac.data_ptr()
            desc.bt = self.bt.data_ptr()
            desc.balpha = self.balpha.data_ptr()
        if self.nonortho:
            desc.alpha_full = self.alpha_full.data_ptr()
            desc.has_cross = int(self.cell_cross)
            if m:
                desc.balpha_row = self.balpha_row.data_ptr()
                desc.bfid = self.bfid.data_ptr()
                desc.finfo = self.finfo.data_ptr()
                desc.nfaces = len(faces)
        if geom_precond not in ("auto", "multigrid", "spectral"):
            raise ValueError(f"geom_precond {geom_precond!r}")
        desc.geom_precond = (
            _lib.PF_GEOM_SPECTRAL
            if geom_precond != "multigrid" and _spectral_allowed(domain, box, sep)
            else _lib.PF_GEOM_MULTIGRID)
        info = getattr(domain, "slab_info", None)
        if info is not None:
            # slab of a larger box (slab.SlabDomain): owned planes between
            # two ghost planes along axis 0
            desc.slab_world, desc.slab_rank = int(info[0]), int(info[1])
            desc.slab_nx, desc.slab_x0 = int(info[2]), int(info[3])
        self.slab = info is not None
        if self.sep_dx is not None and box is not None and \
                not self.nonortho:
            for a in range(d):
                desc.sep_dx[a] = self.sep_dx[a].data_ptr()
                desc.sep_inv[a] = self.sep_inv[a].data_ptr()
        self.comm = None
        self._desc = desc
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.call("pf_plan_create", ctypes.byref(desc), ctypes.byref(handle))
            self.handle = handle
            nbytes = int(_lib.load().pf_workspace_bytes(handle))
            self.workspace = torch.zeros(nbytes, dtype=torch.uint8,
                                         device=device)
            self.mg_bytes = int(_lib.load().pf_mg_workspace_bytes(handle))
            self.mg_levels = int(_lib.load().pf_mg_levels(handle))
            kind = int(_lib.load().pf_mg_kind(handle))
        self.geom_kind = {_lib.PF_GEOM_MULTIGRID: "multigrid",
                          _lib.PF_GEOM_SPECTRAL: "spectral"}.get(kind)
        self.mg_workspace = None
        self._mg_key = None

    def _packed_table(self):
        dom = self.domain
        d, n = dom.dim, dom.n
        nbr, nax, nsg = dom.nbr, dom.nbr_ax, dom.nbr_sign
        table = np.empty((2 * d, n), dtype=np.int64)
        for a in range(d):
            for s in (0, 1):
                nb = nbr[a, s]
                word = (nb | (nax[a, s, :, a].astype(np.int64) << 26)
                        | ((nsg[a, s, :, a] < 0).astype(np.int64) << 28))
                table[2 * a + s] = np.where(nb >= 0, word, 0)
        for f, off in zip(dom.bfaces, self.face_offsets):
            fi = 2 * f.axis + f.side
            table[fi, f.cells] = ~(off + np.arange(f.m, dtype=np.int64))
        missing = np.zeros(n, dtype=bool)
        for fi in range(2 * d):
            a, s = divmod(fi, 2)
            missing |= (nbr[a, s] < 0) & (table[fi] >= 0)
        if missing.any():
            raise ValueError("a cell face has neither a neighbour nor a "
                             "boundary face")
        return table.astype(np.int32)

    # multigrid ----------------------------------------------------------------

    @property
    def has_mg(self):
        return self.mg_bytes > 0

    def mg_prepare(self, k_stencil):
        """Build (or reuse) the multigrid hierarchy for operator K.  The key
        is a per-tensor id plus torch's in-place version counter, so a freed
        and re-allocated tensor at the same address never reuses a stale
        hierarchy."""
        if not self.has_mg:
            return False
        uid = getattr(k_stencil, "_pf_mg_uid", None)
        if uid is None:
            DevicePlan._uid += 1
            uid = DevicePlan._uid
            try:
                k_stencil._pf_mg_uid = uid
            except AttributeError:
                uid = None
        key = (uid, k_stencil._version) if uid is not None else None
        if key is not None and key == self._mg_key:
            return True
        if self.mg_workspace is None:
            self.mg_workspace = torch.empty(self.mg_bytes, dtype=torch.uint8,
                                            device=self.device)
        _lib.call("pf_mg_setup", self.handle, _lib.ptr(k_stencil),
                  _lib.ptr(self.mg_workspace), self.stream)
        self._mg_key = key
        return True

    _uid = 0

    # convenience --------------------------------------------------------------

    @property
    def stream(self):
        return _lib.stream_of(self.device)

    def attach_comm(self, comm):
        """Link this slab plan to the other ranks (slab.SlabComm): from now
        on every entry point on the plan is collective."""
        _lib.call("pf_plan_attach_comm", self.handle, comm.handle,
                  _lib.ptr(self.workspace), self.stream)
        self.comm = comm

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().pf_plan_destroy(h)
            except Exception:
                pass
            self.handle = None
