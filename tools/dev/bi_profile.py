"""Per-pass timing of the batched BiCGStab on the C4 momentum operator
(developer tool): python tools/dev/bi_profile.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2505_16992_b200 import _lib, channel, mesh, piso
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256,192,256").split(","))
dev = torch.device("cuda:0")
dom = mesh.make_channel(shape, ratio=1.03)
u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
plan = dom.device_plan(dev)
c = piso.assemble_momentum(dom, u0, nu, dt)
b = torch.randn((3, dom.n), dtype=torch.float64, device=dev)
n = dom.n
for trans in (0, 1):
    ms = (ctypes.c_double * 5)()
    for rep in range(2):
        _lib.call("pf_bicgstab_profile", plan.handle, _lib.ptr(c), trans, 3, _lib.ptr(b), 8, _lib.ptr(plan.workspace), ms, plan.stream)
    gbs = [200 * n / (ms[0] * 1e6), 128 * n / (ms[1] * 1e6), 200 * n / (ms[2] * 1e6)]
    print(f"trans={trans} tiled={'PF_NO_TILED' not in os.environ} minb={os.environ.get('PF_TILE_MINB','1')} "
          f"pv {ms[0]:.3f} ms ({gbs[0]:.0f} GB/s) st {ms[1]:.3f} ({gbs[1]:.0f}) xr {ms[2]:.3f} ({gbs[2]:.0f}) iter {ms[3]:.3f}", flush=True)
