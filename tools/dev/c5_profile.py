"""Where the C5 LES training step goes (torch.profiler, dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
from paper_2505_16992_b200 import channel, les, mesh, piso, stats as S
dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = os.environ.get("BENCHMARK", "0") == "1"
shape = (64, 48, 64)
dom = mesh.make_channel(shape, ratio=1.095)
state, nu, _ = channel.reichardt_init(dom, 180.0, perturbation=0.1, seed=0, device=dev)
dt = 0.5 * (2 * np.pi / 64) / float(state.u.abs().max())
forcing = channel.WallForcing(dom, dev)
torch.manual_seed(0)
model = les.SGSCorrector(shape, dom.box_layout()[1]).to(dev)
opt = torch.optim.SGD(model.parameters(), lr=1e-3)
bc = torch.cat(list(state.bc), 0)
cfg = piso.StepConfig(dt=dt, nu=nu, tol=1e-8)
u0 = state.u.t().contiguous().t()
sl = S.channel_slices(dom)
ref = tuple(t.detach() for t in S.frame_profile(sl, u0))
tgt = (ref, S.tcf_default_weights(3), sl)
target = state.u[:, 0].reshape(shape).mean(dim=(0, 2)).detach()
for _ in range(3):
    les.train_step(dom, u0, bc, model, opt, forcing, nu, cfg, 16, target, stats_target=tgt)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    les.train_step(dom, u0, bc, model, opt, forcing, nu, cfg, 16, target, stats_target=tgt)
torch.cuda.synchronize()
print("train step ms", (time.perf_counter() - t) / 3 * 1e3, "cudnn.benchmark", torch.backends.cudnn.benchmark)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    les.train_step(dom, u0, bc, model, opt, forcing, nu, cfg, 16, target, stats_target=tgt)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
