"""GPU tier: the production launch settings.  conftest.py turns the solver's
CUDA graphs off and caps the iterations in flight between host polls (for
the in-process multi-slab tests); a fresh process here runs the channel
step and its adjoint with the defaults (graphs on, unbounded batches) and
with the test settings, and the results must agree bitwise (the graphs
replay the same kernels)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2505_16992_b200 import adjoint, channel, mesh, piso
dev = torch.device("cuda:0")
dom = mesh.make_channel((32, 48, 64), ratio=1.03)
u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.3 * (2 * np.pi / 32) / float(u0.abs().max())
g = torch.Generator(device="cpu").manual_seed(0)
w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)
forcing = channel.WallForcing(dom, dev)
ws = piso.PisoWorkspace(dom)
st = piso.make_state(dom, u0=u0, device=dev)
for k in range(3):
    cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(st.u, nu), tol=1e-10)
    tape = piso.StepTape()
    st, dg = piso.piso_step(dom, st, cfg, ws, tape)
    gr = adjoint.backward_step(dom, tape, adjoint.GradState(u=w, p=None), tol=1e-10)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in (st.u, st.p, gr.u):
    h.update(t.contiguous().cpu().numpy().tobytes())
print(json.dumps({"hash": h.hexdigest(), "it": [dg.momentum_iterations, dg.pressure_iterations, gr.solve_iterations]}))
'''


def _run(env_updates, drop, script=SCRIPT):
    env = dict(os.environ)
    env.update(env_updates)
    for k in drop:
        env.pop(k, None)
    out = subprocess.run([sys.executable, "-c", script, ROOT], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


# C1 (32^2 cavity): the whole multigrid V-cycle is one staged single-CTA
# kernel with the CG z-sums folded in (mg.cu k_mg_coarse_staged)
SCRIPT_C1 = r'''
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2505_16992_b200 import adjoint, mesh, piso
dev = torch.device("cuda:0")
dom = mesh.make_cavity((32, 32))
plan = dom.device_plan(dev)
assert plan.geom_kind == "multigrid"
g = torch.Generator(device="cpu").manual_seed(1)
w = torch.randn((dom.n, 2), generator=g, dtype=torch.float64).to(dev)
ws = piso.PisoWorkspace(dom)
st = piso.make_state(dom, u0=np.zeros((dom.n, 2)), device=dev)
for k in range(5):
    cfg = piso.StepConfig(dt=0.02, nu=0.01, tol=1e-10)
    tape = piso.StepTape()
    st, dg = piso.piso_step(dom, st, cfg, ws, tape)
    gr = adjoint.backward_step(dom, tape, adjoint.GradState(u=w, p=None), tol=1e-10)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in (st.u, st.p, gr.u):
    h.update(t.contiguous().cpu().numpy().tobytes())
print(json.dumps({"hash": h.hexdigest(), "it": [dg.momentum_iterations, dg.pressure_iterations, gr.solve_iterations]}))
'''


@pytest.mark.parametrize("script", ["channel", "cavity_c1"])
def test_graphs_and_batches_match_test_settings(script):
    src = SCRIPT if script == "channel" else SCRIPT_C1
    prod = _run({}, ["PF_NO_GRAPHS", "PF_MAX_BATCH"], src)
    test = _run({"PF_NO_GRAPHS": "1", "PF_MAX_BATCH": "4"}, [], src)
    assert prod["it"] == test["it"]
    assert prod["hash"] == test["hash"], "graph replay changed the result"
