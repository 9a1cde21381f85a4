"""ctypes binding of ``libpisob200.so`` (the C ABI in ``include/pisob200.h``).

There is no fallback: if the library is missing or no CUDA device is present
every entry point raises.  All pointers passed are device pointers of torch
tensors; the stream is torch's current stream on the tensors' device.
"""

import ctypes
import threading
import time
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpisob200.so")

c_int = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_ptr = ctypes.c_void_p

PF_TOPO_GATHER = 0
PF_TOPO_BOX = 1
PF_GEOM_NONE = -1
PF_GEOM_MULTIGRID = 0
PF_GEOM_SPECTRAL = 1
PF_BKIND_DIRICHLET = 0
PF_BKIND_OUTFLOW = 1


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("dim", c_int), ("topo", c_int), ("n", c_i64),
        ("box_shape", c_i64 * 3), ("box_periodic", c_int * 3),
        ("box_face_offset", c_i64 * 6),
        ("nbr", c_ptr),
        ("jac", c_ptr), ("tmat", c_ptr), ("alpha_diag", c_ptr),
        ("m", c_i64), ("bcell", c_ptr), ("bface", c_ptr), ("bjac", c_ptr),
        ("bt", c_ptr), ("balpha", c_ptr),
        ("alpha_full", c_ptr), ("balpha_row", c_ptr), ("bfid", c_ptr),
        ("finfo", c_ptr), ("nfaces", c_int), ("has_cross", c_int),
        ("geom_precond", c_int),
        ("slab_world", c_int), ("slab_rank", c_int), ("slab_nx", c_i64),
        ("slab_x0", c_i64),
        ("sep_dx", c_ptr * 3), ("sep_inv", c_ptr * 3), ("ijac", c_ptr),
    ]


class SolverReportC(ctypes.Structure):
    _fields_ = [("converged", c_int), ("iterations", c_int),
                ("residual", c_dbl), ("fallback_used", c_int),
                ("breakdown", c_int)]


# name -> argument types (return type is int32 status unless listed below)
_SIGS = {
    "pf_version": [],
    "pf_launch_count": [],
    "pf_plan_create": [ctypes.POINTER(PlanDesc), ctypes.POINTER(c_ptr)],
    "pf_plan_destroy": [c_ptr],
    "pf_workspace_bytes": [c_ptr],
    "pf_contravariant_flux": [c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_assemble_momentum": [c_ptr, c_ptr, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr],
    "pf_momentum_rhs": [c_ptr, c_ptr, c_ptr, c_ptr, c_int, c_dbl, c_dbl,
                        c_ptr, c_ptr],
    "pf_assemble_pressure": [c_ptr, c_ptr, c_int, c_ptr, c_ptr],
    "pf_h_stage": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_divergence_rhs": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_correct_velocity": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_divergence_max": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                          ctypes.POINTER(c_dbl), c_ptr],
    "pf_divergence_max_dev": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                              c_ptr],
    "pf_stencil_matvec": [c_ptr, c_ptr, c_int, c_int, c_ptr, c_ptr, c_ptr],
    "pf_cg_solve": [c_ptr, c_ptr, c_ptr, c_dbl, c_ptr, c_int, c_dbl, c_int,
                    c_int, c_int, c_ptr, c_ptr, ctypes.POINTER(SolverReportC),
                    c_ptr],
    "pf_mg_workspace_bytes": [c_ptr],
    "pf_mg_levels": [c_ptr],
    "pf_mg_kind": [c_ptr],
    "pf_mg_setup": [c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_bicgstab_solve": [c_ptr, c_ptr, c_int, c_int, c_ptr, c_ptr, c_int,
                          c_dbl, c_int, c_int, c_ptr,
                          ctypes.POINTER(SolverReportC), c_ptr],
    "pf_cg_profile": [c_ptr, c_ptr, c_ptr, c_int, c_int, c_ptr, c_ptr,
                      ctypes.POINTER(c_dbl), c_ptr],
    "pf_slice_moments": [c_ptr, c_ptr, c_int, c_ptr, c_ptr, c_ptr, c_ptr,
                         c_ptr, c_ptr],
    "pf_slice_moments_backward": [c_ptr, c_ptr, c_int, c_ptr, c_ptr, c_ptr,
                                  c_ptr, c_ptr],
    "pf_comm_create": [c_ptr, ctypes.POINTER(c_ptr)],
    "pf_comm_ipc_handle": [c_ptr, c_ptr],
    "pf_comm_open_peer": [c_ptr, c_int, c_ptr],
    "pf_comm_set_local_peer": [c_ptr, c_int, c_ptr],
    "pf_comm_bytes": [c_ptr],
    "pf_plan_attach_comm": [c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_comm_status": [c_ptr, c_ptr],
    "pf_comm_destroy": [c_ptr],
    "pf_halo_exchange": [c_ptr, c_ptr, c_ptr, c_int, c_ptr],
    "pf_comm_allreduce": [c_ptr, c_ptr, c_int, c_int, c_ptr],
    "pf_comm_barrier": [c_ptr, c_ptr],
    "pf_comm_counters": [c_ptr, c_ptr, c_ptr],
    "pf_bicgstab_profile": [c_ptr, c_ptr, c_int, c_int, c_ptr, c_int, c_ptr,
                            ctypes.POINTER(c_dbl), c_ptr],
    "pf_bwd_correct_velocity": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                                c_ptr, c_int, c_ptr, c_ptr],
    "pf_bwd_pressure_outer": [c_ptr, c_ptr, c_ptr, c_ptr, c_int, c_ptr],
    "pf_bwd_pressure_matrix": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_adj_divergence_rhs": [c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr],
    "pf_bwd_h_stage": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                       c_ptr, c_ptr, c_int, c_ptr, c_ptr],
    "pf_bwd_momentum_outer": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_adj_momentum_rhs": [c_ptr, c_ptr, c_ptr, c_dbl, c_dbl, c_ptr, c_ptr,
                            c_ptr, c_int, c_ptr, c_ptr],
    "pf_adj_assemble_momentum": [c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr,
                                 c_ptr],
    "pf_momentum_cross_rhs": [c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr],
    "pf_pressure_cross_rhs": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                              c_ptr],
    "pf_adj_pressure_cross": [c_ptr, c_ptr, c_ptr, c_ptr, c_dbl, c_ptr,
                              c_ptr, c_ptr, c_ptr],
    "pf_adj_momentum_cross": [c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_int,
                              c_ptr, c_ptr, c_ptr],
    "pf_axpy": [c_ptr, c_dbl, c_ptr, c_ptr, c_i64, c_ptr],
    "pf_wide_grad": [c_ptr, c_ptr, c_int, c_ptr, c_ptr, c_ptr],
    "pf_cfl_peak": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "pf_wall_forcing": [c_ptr, c_ptr, c_int, c_ptr, c_ptr, c_ptr, c_ptr,
                        c_int, c_int, c_dbl, c_dbl, c_ptr, c_ptr, c_ptr],
    "pf_wide_grad_adjoint": [c_ptr, c_ptr, c_int, c_ptr, c_ptr, c_ptr],
    "pf_advective_outflow_update": [c_ptr, c_ptr, c_ptr, c_dbl, c_ptr,
                                    ctypes.POINTER(c_dbl), c_ptr],
    "pf_reduce_sum": [c_ptr, c_ptr, c_i64, c_ptr, ctypes.POINTER(c_dbl),
                      c_ptr],
    "pf_reduce_dot": [c_ptr, c_ptr, c_ptr, c_i64, c_ptr,
                      ctypes.POINTER(c_dbl), c_ptr],
    "pf_reduce_maxabs": [c_ptr, c_ptr, c_i64, c_ptr, ctypes.POINTER(c_dbl),
                         c_ptr],
}
_RESTYPES = {"pf_workspace_bytes": c_i64, "pf_mg_workspace_bytes": c_i64,
             "pf_comm_bytes": c_i64, "pf_last_error": ctypes.c_char_p,
             "pf_launch_count": ctypes.c_uint64}

EXPORTED = sorted(list(_SIGS) + ["pf_last_error"])

_lib = None


class LibraryError(RuntimeError):
    pass


def load(path=LIB_PATH):
    """Load and type the library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} is missing: build it with `python -m "
            "paper_2505_16992_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    lib.pf_last_error.restype = ctypes.c_char_p
    lib.pf_last_error.argtypes = []
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


# diagnosis: a list here collects (entry point, host start, host end,
# device start event, device end event) of every call (tools/dev/trace.py)
TRACE = None


def call(name, *args):
    """Invoke an entry point; non-zero status raises LibraryError.  The
    tensors whose pointers were taken for this call (ptr) stay referenced
    until it has enqueued its work: a temporary such as ``ptr(soa(h))``
    would otherwise return its block to the caching allocator before the
    call, and the next temporary of the same argument list could reuse
    (and overwrite) it ahead of the kernel in stream order."""
    lib = load()
    tr = TRACE
    if tr is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
    try:
        rc = getattr(lib, name)(*args)
    finally:
        _keep.refs = []
    if tr is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        tr.append((name, h0, time.perf_counter(), e0, e1))
    if rc != 0:
        msg = lib.pf_last_error().decode(errors="replace")
        raise LibraryError(f"{name} failed (status {rc}): {msg}")
    return rc


def require_cuda(device):
    if device.type != "cuda" or not torch.cuda.is_available():
        raise LibraryError(
            "the PISO step runs only on a CUDA device (sm_100a); "
            "there is no CPU fallback")


_keep = threading.local()


def ptr(t):
    """Device pointer of a tensor (None -> NULL); the tensor is kept alive
    until the next call() returns (per host thread)."""
    if t is None:
        return None
    refs = getattr(_keep, "refs", None)
    if refs is None:
        refs = _keep.refs = []
    refs.append(t)
    return c_ptr(t.data_ptr())


class nvtx:
    """NVTX range around a stage (SURVEY §5 tracing): visible in nsys /
    ncu --nvtx timelines; PF_NVTX=0 turns the ranges off."""
    on = os.environ.get("PF_NVTX", "1") != "0"

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if nvtx.on:
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if nvtx.on:
            torch.cuda.nvtx.range_pop()
        return False


def stream_of(device):
    return c_ptr(torch.cuda.current_stream(device).cuda_stream)
