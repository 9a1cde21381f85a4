"""Spectral pressure-CG iteration on the C4 operator under ncu (dev tool)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2505_16992_b200 import _lib, channel, mesh, piso
dev = torch.device("cuda:0")
shape = (256, 192, 256)
dom = mesh.make_channel(shape, ratio=1.03)
u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.3 * (2 * np.pi / 256) / float(u0.abs().max())
plan = dom.device_plan(dev)
c = piso.assemble_momentum(dom, u0, nu, dt)
k = torch.empty_like(c)
_lib.call("pf_assemble_pressure", plan.handle, _lib.ptr(c), 0, _lib.ptr(k), plan.stream)
plan.mg_prepare(k)
b = torch.randn(dom.n, dtype=torch.float64, device=dev)
ms = (ctypes.c_double * 12)()
_lib.call("pf_cg_profile", plan.handle, _lib.ptr(k), _lib.ptr(b), 4, 2, _lib.ptr(plan.workspace), _lib.ptr(plan.mg_workspace), ms, plan.stream)
print([round(v, 4) for v in ms])
