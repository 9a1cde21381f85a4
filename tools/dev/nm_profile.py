"""Neumann-2 BiCGStab passes on the C4 momentum operator (developer tool):
per-pass CUDA-event timing via pf_bicgstab_profile; under ncu, capture with
-k regex:k_bi_nm.   python tools/dev/nm_profile.py [shape] [trans]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2505_16992_b200 import _lib, channel, mesh, piso
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256,192,256").split(","))
transes = [int(sys.argv[2])] if len(sys.argv) > 2 else [0, 1]
iters = int(os.environ.get("NM_ITERS", "8"))
dev = torch.device("cuda:0")
dom = mesh.make_channel(shape, ratio=1.03)
u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
plan = dom.device_plan(dev)
c = piso.assemble_momentum(dom, u0, nu, dt)
b = torch.randn((3, dom.n), dtype=torch.float64, device=dev)
n = dom.n
for trans in transes:
    ms = (ctypes.c_double * 5)()
    for rep in range(int(os.environ.get("NM_REPS", "2"))):
        _lib.call("pf_bicgstab_profile", plan.handle, _lib.ptr(c), trans, 3, _lib.ptr(b), iters, _lib.ptr(plan.workspace), ms, plan.stream)
    gbs = [200 * n / (ms[0] * 1e6), 128 * n / (ms[1] * 1e6), 192 * n / (ms[2] * 1e6)]
    print(f"trans={trans} precond={int(ms[4])} pv {ms[0]*1e3:.1f} us ({gbs[0]:.0f} GB/s) st {ms[1]*1e3:.1f} ({gbs[1]:.0f}) "
          f"xr {ms[2]*1e3:.1f} ({gbs[2]:.0f}) iter {ms[3]*1e3:.1f}", flush=True)
