"""GPU tier: the slab path across PROCESSES, through CUDA-IPC-mapped peer
buffers -- the exact mechanism of one process per GPU on an NVSwitch box,
here with both processes on the one B200 (their kernels time-slice, so this
is a correctness test, not a timing).  Process group: gloo on 127.0.0.1
(handles and the final comparison only)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, production=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      CUDA_MODULE_LOADING="EAGER", PF_COMM_TIMEOUT_S="30")
    if production:
        # one process per GPU in production: the solver's CUDA graphs and
        # unbounded batches between polls (conftest limits them for the
        # in-process slab tests only)
        os.environ.pop("PF_NO_GRAPHS", None)
        os.environ.pop("PF_MAX_BATCH", None)
    import torch.distributed as dist
    from paper_2505_16992_b200 import adjoint, channel, mesh, piso, slab
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dom = mesh.make_channel((8, 12, 8), ratio=1.1)
    u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=0, device=dev)
    dt = 0.3 * (2 * np.pi / 8) / float(u0.abs().max())
    g = torch.Generator(device="cpu").manual_seed(1)
    w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)
    src = torch.tensor([1e-3, 0.0, 0.0], dtype=torch.float64, device=dev)
    sd = slab.SlabDomain(dom, rank, world)
    comm = slab.SlabComm.distributed(sd, dev)
    st = piso.make_state(sd, u0=sd.scatter(u0), device=dev)
    cfg = piso.StepConfig(dt=dt, nu=nu, source=src, tol=1e-12)
    tape = piso.StepTape()
    new, diag = piso.piso_step(sd, st, cfg, None, tape)
    gr = adjoint.backward_step(sd, tape, adjoint.GradState(
        u=sd.scatter(w), p=torch.zeros(sd.n, dtype=torch.float64,
                                       device=dev)), tol=1e-12)
    torch.cuda.synchronize()
    comm.status()
    u_own = sd.owned(new.u).cpu().contiguous()
    g_own = sd.owned(gr.u).cpu().contiguous()
    us = [torch.empty_like(u_own) for _ in range(world)]
    gs = [torch.empty_like(g_own) for _ in range(world)]
    dist.all_gather(us, u_own)
    dist.all_gather(gs, g_own)
    if rank == 0:
        ref_state = piso.make_state(dom, u0=u0, device=dev)
        tape0 = piso.StepTape()
        ref, _ = piso.piso_step(dom, ref_state, cfg, None, tape0)
        gref = adjoint.backward_step(dom, tape0, adjoint.GradState(
            u=w, p=torch.zeros(dom.n, dtype=torch.float64, device=dev)),
            tol=1e-12)
        u = torch.cat(us).numpy()
        gu = torch.cat(gs).numpy()
        ru, rg = ref.u.cpu().numpy(), gref.u.cpu().numpy()
        np.savez(out_path, eu=np.abs(u - ru).max() / np.abs(ru).max(),
                 eg=np.abs(gu - rg).max() / np.abs(rg).max(),
                 nu_slab=gr.nu, nu_ref=gref.nu)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("production", [False, True])
def test_slab_step_across_processes_ipc(tmp_path, production):
    import torch.multiprocessing as mp
    out = str(tmp_path / "ipc.npz")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out, production))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    assert not alive, "slab processes hung"
    assert all(p.exitcode == 0 for p in procs)
    r = np.load(out)
    assert float(r["eu"]) < 1e-8
    assert float(r["eg"]) < 1e-8
    assert float(r["nu_slab"]) == pytest.approx(float(r["nu_ref"]), rel=1e-8)
