"""GPU tier: the slab-decomposed step (SURVEY.md §8 e) against the
single-domain step on the same inputs.

Several slabs run in ONE process on one B200, each on its own CUDA stream
and host thread, linked through the same peer-memory communicator the
multi-GPU path uses (here the peers' buffers are same-device pointers
instead of CUDA-IPC mappings).  Halo exchange, the in-kernel cross-rank
reductions and the spectral preconditioner's all-to-all transposes all run
exactly as on 8 GPUs; only the summation order of the global reductions
differs from the single-domain run, so fields and gradients agree to solver
tolerance, not bitwise.
"""

import os
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-12
FIELD_TOL = 1e-8


def _rel(a, b):
    a = a.detach().cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.detach().cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _setup(shape=(8, 12, 8), ratio=1.1):
    from paper_2505_16992_b200 import channel, mesh
    dev = torch.device("cuda:0")
    dom = mesh.make_channel(shape, ratio=ratio)
    u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=0, device=dev)
    dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
    g = torch.Generator(device="cpu").manual_seed(1)
    w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)
    return dom, dev, u0, nu, dt, w


def _single(dom, dev, u0, nu, dt, w, steps=1):
    from paper_2505_16992_b200 import adjoint, channel, piso
    st = piso.make_state(dom, u0=u0, device=dev)
    forcing = channel.WallForcing(dom, dev)
    ws = piso.PisoWorkspace(dom)
    out = []
    for _ in range(steps):
        cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(st.u, nu), tol=TOL)
        tape = piso.StepTape()
        st, diag = piso.piso_step(dom, st, cfg, ws, tape)
        g = adjoint.backward_step(dom, tape, adjoint.GradState(
            u=w, p=torch.zeros(dom.n, dtype=torch.float64, device=dev)),
            tol=TOL)
        out.append((st, diag, g))
    torch.cuda.synchronize()
    return out


def _slabs(dom, dev, u0, nu, dt, w, world, steps=1):
    """Run `world` slabs in threads; returns per-rank [(state, diag, grad)]
    and the slab domains."""
    from paper_2505_16992_b200 import adjoint, piso, slab
    slabs = [slab.SlabDomain(dom, r, world) for r in range(world)]
    comms = slab.SlabComm.local_group(slabs, dev)
    results = [None] * world
    errors = []
    ready = threading.Barrier(world)

    def work(r):
        try:
            sd = slabs[r]
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                _prewarm(ready)
                st = piso.make_state(sd, u0=sd.scatter(u0), device=dev)
                forcing = slab.SlabWallForcing(sd, dev)
                ws = piso.PisoWorkspace(sd)
                wl = sd.scatter(w)
                out = []
                for _ in range(steps):
                    cfg = piso.StepConfig(dt=dt, nu=nu,
                                          source=forcing(st.u, nu), tol=TOL)
                    tape = piso.StepTape()
                    st, diag = piso.piso_step(sd, st, cfg, ws, tape)
                    g = adjoint.backward_step(sd, tape, adjoint.GradState(
                        u=wl, p=torch.zeros(sd.n, dtype=torch.float64,
                                            device=dev)), tol=TOL)
                    out.append((st, diag, g))
                s.synchronize()
                comms[r].status()
                results[r] = out
        except Exception as exc:  # surfaced in the main thread
            errors.append((r, exc))

    # the inputs were written on the default stream; the slab streams start
    # from a synchronised device
    torch.cuda.synchronize()
    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in threads), "slab threads hung"
    if errors:
        raise errors[0][1]
    return slabs, results


def _prewarm(barrier, nbytes=256 << 20):
    """Reserve this thread's stream a block of the caching allocator, then
    wait for every slab thread.  A cudaMalloc synchronises the whole device:
    issued while another slab's kernel spins on this slab's next step it
    would deadlock (one process per GPU never shares a device this way)."""
    big = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    # and a segment of the small-block pool (< 1 MB allocations)
    small = [torch.empty(4096, dtype=torch.uint8, device="cuda:0")
             for _ in range(256)]
    del big, small
    torch.cuda.current_stream().synchronize()
    barrier.wait(timeout=120)


def _gather(slabs, results, k, pick, dom_n, ncol):
    out = np.zeros((dom_n, ncol)) if ncol else np.zeros(dom_n)
    for sd, res in zip(slabs, results):
        v = pick(res[k])
        v = v.detach().cpu().numpy() if torch.is_tensor(v) else v
        sd.gather_into(v.reshape(sd.n, -1) if ncol else v.reshape(sd.n), out)
    return out


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_step_matches_single_domain(world):
    dom, dev, u0, nu, dt, w = _setup()
    ref = _single(dom, dev, u0, nu, dt, w, steps=2)
    slabs, res = _slabs(dom, dev, u0, nu, dt, w, world, steps=2)
    for k in range(2):
        st, diag, g = ref[k]
        u = _gather(slabs, res, k, lambda r: r[0].u, dom.n, 3)
        p = _gather(slabs, res, k, lambda r: r[0].p, dom.n, 0)
        gu = _gather(slabs, res, k, lambda r: r[2].u, dom.n, 3)
        assert _rel(u, st.u) < FIELD_TOL
        assert _rel(p, st.p) < FIELD_TOL
        assert _rel(gu, g.u) < FIELD_TOL
        for r in range(world):
            assert res[r][k][2].nu == pytest.approx(g.nu, rel=FIELD_TOL)
            # every rank took the same global decisions
            assert res[r][k][1].pressure_iterations == \
                res[0][k][1].pressure_iterations
            assert res[r][k][2].nu == res[0][k][2].nu
        # iteration counts: same solver, same global operator
        assert abs(res[0][k][1].pressure_iterations
                   - diag.pressure_iterations) <= 2
        assert abs(res[0][k][1].momentum_iterations
                   - diag.momentum_iterations) <= 3


@pytest.mark.parametrize("shape", [(8, 8, 256), (256, 8, 8)])
def test_slab_step_256_point_transforms(shape):
    """Length-256 Z / X: the register four-step FFT kernels of the spectral
    preconditioner in their slab form (transposes over peer memory)."""
    dom, dev, u0, nu, dt, w = _setup(shape)
    ref = _single(dom, dev, u0, nu, dt, w, steps=1)
    slabs, res = _slabs(dom, dev, u0, nu, dt, w, 2, steps=1)
    st, diag, g = ref[0]
    u = _gather(slabs, res, 0, lambda r: r[0].u, dom.n, 3)
    p = _gather(slabs, res, 0, lambda r: r[0].p, dom.n, 0)
    gu = _gather(slabs, res, 0, lambda r: r[2].u, dom.n, 3)
    assert _rel(u, st.u) < FIELD_TOL
    assert _rel(p, st.p) < FIELD_TOL
    assert _rel(gu, g.u) < FIELD_TOL


def test_slab_wall_forcing_matches_global():
    from paper_2505_16992_b200 import channel, slab
    dom, dev, u0, nu, dt, w = _setup()
    ref = channel.WallForcing(dom, dev)(u0, nu)
    slabs = [slab.SlabDomain(dom, r, 2) for r in range(2)]
    slab.SlabComm.local_group(slabs, dev)
    out = [None, None]
    ready = threading.Barrier(2)

    def work(r):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            _prewarm(ready)
            out[r] = slab.SlabWallForcing(slabs[r], dev)(
                slabs[r].scatter(u0), nu)
            s.synchronize()

    torch.cuda.synchronize()
    ts = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    for r in range(2):
        assert _rel(out[r], ref) < 1e-13


def test_slab_halo_and_allreduce_primitives():
    """pf_halo_exchange / pf_comm_allreduce on 3 slabs: ghost planes equal
    the neighbours' edge planes (ring), sums equal the global sum."""
    from paper_2505_16992_b200 import mesh, slab
    dev = torch.device("cuda:0")
    dom = mesh.make_channel((6, 4, 4), ratio=1.1)
    slabs = [slab.SlabDomain(dom, r, 3) for r in range(3)]
    slab.SlabComm.local_group(slabs, dev)
    glob = torch.arange(dom.n * 2, dtype=torch.float64,
                        device=dev).reshape(2, dom.n)
    fields, sums = [], []
    for sd in slabs:
        f = torch.full((2, sd.n), -1.0, dtype=torch.float64, device=dev)
        own = sd.owned_global_rows()
        f[:, sd.owned_slice] = glob[:, torch.as_tensor(own, device=dev)]
        fields.append(f)
        sums.append(torch.tensor([float(sd.rank + 1), -float(sd.rank)],
                                 dtype=torch.float64, device=dev))

    ready = threading.Barrier(3)

    def work(r):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            _prewarm(ready)
            plan = slabs[r].device_plan(dev)
            slab.halo_exchange(plan, fields[r])
            slab.allreduce_(plan, sums[r])
            s.synchronize()

    torch.cuda.synchronize()
    ts = [threading.Thread(target=work, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    for sd, f, sm in zip(slabs, fields, sums):
        rows = torch.as_tensor(sd._global_rows(), device=dev)
        assert torch.equal(f, glob[:, rows])
        assert sm.tolist() == [6.0, -3.0]
