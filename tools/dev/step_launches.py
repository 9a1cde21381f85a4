"""One C4 fwd+adjoint step between cudaProfilerStart/Stop (developer tool):
ncu --profile-from-start off --metrics gpu__time_duration.sum ... python
tools/dev/step_launches.py [shape]  -> the step's launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2505_16992_b200 import adjoint, channel, mesh, piso
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256,192,256").split(","))
dev = torch.device("cuda:0")
dom = mesh.make_channel(shape, ratio=1.03)
u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
g = torch.Generator(device="cpu").manual_seed(0)
w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)
cot = adjoint.GradState(u=w, p=torch.zeros(dom.n, dtype=torch.float64, device=dev))
forcing = channel.WallForcing(dom, dev)
ws = piso.PisoWorkspace(dom)
state = piso.make_state(dom, u0=u0, device=dev)


def step(state):
    cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(state.u, nu), tol=1e-8)
    tape = piso.StepTape()
    new, dg = piso.piso_step(dom, state, cfg, ws, tape)
    gr = adjoint.backward_step(dom, tape, cot, tol=1e-8)
    return new, dg, gr


for _ in range(3):
    state, dg, gr = step(state)
torch.cuda.synchronize()
torch.cuda.profiler.start()
state, dg, gr = step(state)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", dg.momentum_iterations, dg.pressure_iterations, gr.solve_iterations)
