"""Slab decomposition of a single-box domain across GPUs (SURVEY.md §8 e).

The 3D channel (C4) is split along its periodic streamwise axis 0 into
``world`` slabs, one per rank (one process per GPU).  Rank ``r`` owns
``nxl`` consecutive planes and holds them between two ghost planes that
mirror the neighbouring ranks' edge planes, so its local mesh is a box of
``nxl + 2`` planes (:class:`SlabDomain`, a :class:`~.mesh.Domain`).  The
step code is unchanged: ``piso.piso_step`` and ``adjoint.backward_step`` run
on the slab domain, and the C library exchanges ghost planes and reduces
across ranks inside its entry points (include/pisob200.h, "slab
decomposition"):

* ghost planes move by peer-memory stores (NVLink P2P through CUDA IPC, or
  direct pointers when several slabs share one device in a test),
* solver dot products and means are reduced across ranks inside the
  kernels that form them (the last CTA of each fused reduction stores its
  partial totals into every peer's slot and sums the slots in rank order),
* the spectral pressure preconditioner transposes its spectrum across ranks
  (kz-slabs after the Z transform) by direct peer stores and loads.

So forward+adjoint steps on ``world`` slabs reproduce the single-GPU step up
to the summation order of the global reductions.

Typical use (one process per GPU under torchrun)::

    dom = mesh.make_channel((256, 192, 256), ratio=1.03)
    sd = slab.SlabDomain(dom, rank, world)
    comm = slab.SlabComm.distributed(sd, device)    # IPC handles via
                                                    # torch.distributed
    state = sd.scatter_state(global_state)          # or sd.local_state(u)
    new, diag = piso.piso_step(sd, state, cfg, ws, tape)

Fields of a slab are (n_local, d) with n_local = (nxl + 2) * plane; use
:meth:`SlabDomain.owned` for the owned part and :meth:`SlabDomain.scatter`
/ :meth:`SlabDomain.gather` to move between global and local layouts.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .mesh import BlockSpec, Dirichlet, Domain, _grid_vertices, _self_periodic


def slab_bounds(nx, rank, world):
    """(x0, nxl): the planes rank `rank` owns of `nx` split over `world`
    ranks (the first nx % world ranks take one more)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside 0..{world - 1}")
    base, rem = divmod(int(nx), int(world))
    nxl = base + (1 if rank < rem else 0)
    x0 = rank * base + min(rank, rem)
    return x0, nxl


class SlabDomain(Domain):
    """Rank `rank`'s slab (with one ghost plane per side) of a single-block
    domain whose axis 0 is periodic.  The boundary faces of the other axes
    must be periodic or Dirichlet with a uniform value (the channel walls)."""

    def __init__(self, domain, rank, world):
        box = domain.box_layout()
        if box is None:
            raise ValueError("slab decomposition needs a single-block box")
        shape, periodic = box
        if not periodic[0]:
            raise ValueError("slab decomposition needs a periodic axis 0 "
                             "(the ranks form a ring)")
        coords = domain._separable[0]
        if coords is None:
            raise ValueError("slab decomposition needs a tensor-product grid")
        nx = shape[0]
        x0, nxl = slab_bounds(nx, rank, world)
        if nxl < 1:
            raise ValueError(f"{world} ranks leave rank {rank} no plane of "
                             f"{nx}")
        d = domain.dim
        # local vertices: global planes x0 - 1 .. x0 + nxl, wrapped
        # periodically (the ghost cells are copies of the neighbours' cells)
        xv = np.asarray(coords[0], dtype=np.float64)
        widths = np.diff(xv)
        idx = np.arange(x0 - 1, x0 + nxl + 1)
        w = widths[idx % nx]
        # vertex 0 of the local box is the left face of global plane x0 - 1
        left = xv[x0] - w[0]
        local_x = np.concatenate([[left], left + np.cumsum(w)])
        blk = BlockSpec(_grid_vertices(local_x, *coords[1:]))
        bnd = {(0, 0, 0): _self_periodic(0, 0, 1, d),
               (0, 0, 1): _self_periodic(0, 0, 0, d)}
        for a in range(1, d):
            for s in (0, 1):
                spec = domain.boundaries[(0, a, s)]
                if isinstance(spec, Dirichlet):
                    if np.ndim(spec.value) > 1:
                        raise ValueError("slab decomposition supports "
                                         "uniform Dirichlet values only")
                    bnd[(0, a, s)] = spec
                elif periodic[a]:
                    bnd[(0, a, s)] = _self_periodic(0, a, 1 - s, d)
                else:
                    raise ValueError(f"boundary {(0, a, s)} of kind "
                                     f"{type(spec).__name__} is not "
                                     "supported on a slab")
        super().__init__([blk], bnd)
        self.global_domain = domain
        self.rank, self.world = int(rank), int(world)
        self.x0, self.nxl, self.nx = int(x0), int(nxl), int(nx)
        self.plane = int(np.prod(shape[1:]))
        self.global_shape = tuple(shape)
        # consumed by DevicePlan (pf_plan_desc.slab_*)
        self.slab_info = (self.world, self.rank, self.nx, self.x0)

    # -- layout helpers ------------------------------------------------------

    @property
    def owned_slice(self):
        return slice(self.plane, self.plane * (self.nxl + 1))

    def owned(self, field):
        """Owned rows of an (n_local, ...) field (a view)."""
        return field[self.owned_slice]

    def _global_rows(self):
        """Global cell index of every local row (ghost rows wrap)."""
        xs = (np.arange(self.x0 - 1, self.x0 + self.nxl + 1) % self.nx)
        return (xs[:, None] * self.plane
                + np.arange(self.plane)[None, :]).reshape(-1)

    def scatter(self, field):
        """Local (n_local, ...) copy of a global (n, ...) field, ghost planes
        included (torch tensor or NumPy array)."""
        rows = self._global_rows()
        if torch.is_tensor(field):
            return field[torch.as_tensor(rows, device=field.device)]
        return np.asarray(field)[rows]

    def owned_global_rows(self):
        return np.arange(self.x0 * self.plane,
                         (self.x0 + self.nxl) * self.plane)

    def gather_into(self, field, out):
        """Write the owned rows of a local field into a global array."""
        sl = slice(self.x0 * self.plane, (self.x0 + self.nxl) * self.plane)
        out[sl] = self.owned(field)
        return out

    def local_bc(self, global_bc):
        """Per-face boundary values of this slab from the global domain's
        per-face list (the faces of axes >= 1 restricted to the local
        planes, ghost planes included)."""
        g = self.global_domain
        out = []
        gfaces = {(f.axis, f.side): (f, v) for f, v in zip(g.bfaces,
                                                          global_bc)}
        for f in self.bfaces:
            gf, val = gfaces[(f.axis, f.side)]
            # a face of axis a >= 1 is an area grid whose first axis is X
            area = gf.area_shape
            v = val.reshape(tuple(area) + (val.shape[-1],)) \
                if hasattr(val, "reshape") else np.asarray(val)
            xs = np.arange(self.x0 - 1, self.x0 + self.nxl + 1) % self.nx
            if torch.is_tensor(v):
                loc = v[torch.as_tensor(xs, device=v.device)]
            else:
                loc = v[xs]
            out.append(loc.reshape(-1, val.shape[-1]))
        return out

    def scatter_state(self, state):
        """FlowState of this slab from a global FlowState."""
        from .piso import FlowState
        u = state.u
        u_loc = self.scatter(u.contiguous() if torch.is_tensor(u) else u)
        p_loc = self.scatter(state.p)
        if torch.is_tensor(u_loc):
            u_loc = u_loc.t().contiguous().t()
        return FlowState(u=u_loc, p=p_loc, bc=self.local_bc(state.bc),
                         t=state.t, step=state.step)


class SlabComm:
    """This rank's communicator (symmetric peer-memory buffer) for a slab
    plan.  Build with :meth:`local_group` (several slabs in one process on
    one device) or :meth:`distributed` (one process per GPU)."""

    def __init__(self, plan):
        self.plan = plan
        h = ctypes.c_void_p()
        with torch.cuda.device(plan.device):
            _lib.call("pf_comm_create", plan.handle, ctypes.byref(h))
        self.handle = h

    def ipc_handle(self):
        buf = (ctypes.c_char * 64)()
        _lib.call("pf_comm_ipc_handle", self.handle, buf)
        return bytes(buf)

    def counters(self):
        """(allreduce, halo, barrier, vector allreduce) sequence numbers."""
        out = (ctypes.c_uint64 * 4)()
        _lib.call("pf_comm_counters", self.handle, out, self.plan.stream)
        return tuple(int(v) for v in out)

    def status(self):
        _lib.call("pf_comm_status", self.handle, self.plan.stream)

    @classmethod
    def local_group(cls, slabs, device):
        """Communicators for slab domains of one process on one device
        (slabs[q].rank == q); attaches them to the slabs' plans."""
        plans = [sd.device_plan(device) for sd in slabs]
        comms = [cls(p) for p in plans]
        for c in comms:
            for q, o in enumerate(comms):
                if o is not c:
                    _lib.call("pf_comm_set_local_peer", c.handle, q, o.handle)
        for p, c in zip(plans, comms):
            p.attach_comm(c)
        return comms

    @classmethod
    def distributed(cls, slab, device, group=None):
        """This rank's communicator; the peers' buffers are mapped through
        CUDA IPC handles exchanged with torch.distributed (any backend)."""
        import torch.distributed as dist
        plan = slab.device_plan(device)
        comm = cls(plan)
        handles = [None] * slab.world
        dist.all_gather_object(handles, comm.ipc_handle(), group=group)
        for q, hnd in enumerate(handles):
            if q != slab.rank:
                buf = ctypes.create_string_buffer(hnd, 64)
                _lib.call("pf_comm_open_peer", comm.handle, q, buf)
        # every rank has mapped every buffer before anyone writes into one
        dist.barrier(group=group)
        plan.attach_comm(comm)
        return comm

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().pf_comm_destroy(h)
            except Exception:
                pass
            self.handle = None


def allreduce_(plan, t, op="sum"):
    """In-place sum / max of a float64 device tensor over the slab ranks
    (no-op on a plan without a communicator)."""
    if getattr(plan, "comm", None) is None:
        return t
    assert t.dtype == torch.float64 and t.is_contiguous()
    _lib.call("pf_comm_allreduce", plan.handle, _lib.ptr(t), t.numel(),
              0 if op == "sum" else 1, plan.stream)
    return t


def halo_exchange(plan, *arrays):
    """Refresh the ghost planes of (k, n) / (n,) float64 device arrays."""
    if getattr(plan, "comm", None) is None:
        return
    ptrs = (ctypes.c_uint64 * len(arrays))(*[a.data_ptr() for a in arrays])
    nc = (ctypes.c_int32 * len(arrays))(
        *[1 if a.dim() == 1 else a.shape[0] for a in arrays])
    _lib.call("pf_halo_exchange", plan.handle, ptrs, nc, len(arrays),
              plan.stream)


class SlabWallForcing:
    """channel.WallForcing on a slab: the per-wall sums of u/dist over the
    rank's owned wall cells, added over the ranks inside the fused kernel's
    reduction and divided by the global row sizes (S/piso.py:523-542)."""

    def __init__(self, slab, device, wall_axis=1, flow_axis=0, delta=1.0):
        from .channel import WallForcing
        lo, hi = slab.plane, slab.plane * (slab.nxl + 1)
        # the global row size of each wall: its owned cells x nx / nxl
        probe = WallForcing(slab, device, wall_axis, flow_axis, delta,
                            owned=(lo, hi))
        owned = np.diff(probe.seg.cpu().numpy())
        counts = [float(slab.nx * int(k) // max(slab.nxl, 1)) for k in owned]
        self._wf = WallForcing(slab, device, wall_axis, flow_axis, delta,
                               owned=(lo, hi), counts=counts)

    def __call__(self, u, nu):
        return self._wf(u, nu)


__all__ = ["slab_bounds", "SlabDomain", "SlabComm", "SlabWallForcing",
           "allreduce_", "halo_exchange"]
