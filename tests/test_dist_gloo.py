"""CPU tier, world_size 2 (gloo): the data-parallel host logic of the LES
training step (config 5) -- each rank rolls out its own sample, the CNN
gradients are averaged with one all-reduce, and both ranks end with the
parameters a single process gets from the averaged gradient.  The PISO step
is replaced by a differentiable CPU stand-in (the real step needs a GPU);
this tests the decomposition and collective, not the solver."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_16992_b200 import les

SHAPE = (4, 6, 4)


def _stand_in(u, src):
    return u + 0.1 * (src - 0.05 * u)


def _forcing(u, nu):
    return torch.zeros(3, dtype=torch.float64)


def _setup(rank):
    torch.manual_seed(0)
    model = les.SGSCorrector(SHAPE, (True, False, True), width=4, scale=0.5)
    g = torch.Generator().manual_seed(100 + rank)
    n = SHAPE[0] * SHAPE[1] * SHAPE[2]
    u0 = torch.randn((n, 3), generator=g, dtype=torch.float64)
    target = torch.linspace(0.0, 1.0, SHAPE[1], dtype=torch.float64)
    return model, u0, target


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, u0, target = _setup(rank)
    opt = torch.optim.SGD(model.parameters(), lr=0.1)
    loss = les.train_step(None, u0, None, model, opt, _forcing, 0.01, None,
                          3, target, step_fn=_stand_in)
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
    out[rank] = (loss, flat)
    dist.destroy_process_group()


def test_data_parallel_gradient_average_world2():
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    # single-process reference: average of the two ranks' gradients
    grads = []
    for rank in range(2):
        model, u0, target = _setup(rank)
        loss, _ = les.unrolled_loss(None, u0, None, model, _forcing, 0.01,
                                    None, 3, target, step_fn=_stand_in)
        loss.backward()
        grads.append([p.grad.clone() for p in model.parameters()])
        assert out[rank][0] == pytest.approx(float(loss), rel=1e-12)
    model, _, _ = _setup(0)
    with torch.no_grad():
        for p, g0, g1 in zip(model.parameters(), grads[0], grads[1]):
            p -= 0.1 * 0.5 * (g0 + g1)
    ref = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
    assert torch.allclose(out[0][1], out[1][1], rtol=0, atol=0)
    assert torch.allclose(out[0][1], ref, rtol=1e-12, atol=1e-14)
