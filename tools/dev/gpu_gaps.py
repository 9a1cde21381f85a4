"""GPU idle gaps inside one C4 fwd+adjoint step (developer tool): the CUDA
kernel timeline of the step from torch.profiler (CUPTI), the idle time
between consecutive kernels, and the largest gaps with their neighbours.
    python tools/dev/gpu_gaps.py [shape] > gpurun_out/gaps.txt"""
import json, os, sys, tempfile
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
    return new


for _ in range(3):
    state = step(state)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        state = step(state)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0, t1 = k[0]["ts"], k[-1]["ts"] + k[-1]["dur"]
busy = sum(e["dur"] for e in k)
gaps = []
for a, b in zip(k, k[1:]):
    gap = b["ts"] - (a["ts"] + a["dur"])
    if gap > 0:
        gaps.append((gap, a["name"][:60], b["name"][:60]))
tot_gap = sum(g_[0] for g_ in gaps)
print(f"2 steps: span {(t1 - t0)/1e3:.2f} ms, kernels busy {busy/1e3:.2f} ms, idle {tot_gap/1e3:.2f} ms, {len(k)} GPU ops")
import collections
by = collections.Counter()
for gap, a, b in gaps:
    by[(a.split("(")[0][-40:], b.split("(")[0][-40:])] += gap
for (a, b), gsum in by.most_common(25):
    print(f"{gsum/1e3:7.3f} ms  after {a:40s} before {b}")
