"""GPU tier: the 2.5D-tiled BiCGStab stencil passes (3D boxes whose Y / Z
extents are whole 8 x 32 tiles) against the generic gather kernels
(PF_NO_TILED=1) and against an exact sparse solve of the same system."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _system(shape, seed=0):
    from paper_2505_16992_b200 import channel, mesh, piso
    dev = torch.device("cuda:0")
    dom = mesh.make_channel(shape, ratio=1.1)
    u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=seed, device=dev)
    dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
    c = piso.assemble_momentum(dom, u0, nu, dt)
    g = torch.Generator(device="cpu").manual_seed(seed)
    b = torch.randn((3, dom.n), generator=g, dtype=torch.float64).to(dev)
    return dom, c, b


def _solve(dom, c, b, transpose, tiled, tol=1e-12, precond="jacobi"):
    """Jacobi by default: the generic kernels run Jacobi, so iteration counts
    compare one to one (the Neumann-2 passes: test_gpu_neumann.py)."""
    from paper_2505_16992_b200 import linalg
    plan = dom.device_plan(b.device)
    if tiled:
        os.environ.pop("PF_NO_TILED", None)
    else:
        os.environ["PF_NO_TILED"] = "1"
    try:
        x, reps = linalg.bicgstab_solve(plan, c, b, tol=tol,
                                        transpose=transpose, precond=precond)
    finally:
        os.environ.pop("PF_NO_TILED", None)
    torch.cuda.synchronize()
    return x, reps


@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("shape", [(8, 16, 32), (12, 8, 64)])
def test_tiled_bicgstab_matches_generic_and_exact(shape, transpose):
    from paper_2505_16992_b200 import linalg
    dom, c, b = _system(shape)
    xt, rt = _solve(dom, c, b, transpose, tiled=True)
    xg, rg = _solve(dom, c, b, transpose, tiled=False)
    assert [r.iterations for r in rt] == [r.iterations for r in rg]
    scale = float(xg.abs().max())
    assert float((xt - xg).abs().max()) / scale < 1e-10
    import scipy.sparse.linalg as sla
    a = linalg.stencil_to_csr(dom, c)
    a = a.T.tocsc() if transpose else a.tocsc()
    lu = sla.splu(a)
    for q in range(3):
        ex = lu.solve(b[q].cpu().numpy())
        assert np.abs(xt[q].cpu().numpy() - ex).max() / np.abs(ex).max() \
            < 1e-9


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("precond", ["jacobi", "neumann2"])
def test_tiled_slab_matches_single_domain(precond, world):
    """The tiled passes on slab plans (ghost planes as the X neighbours;
    Neumann-2: the edge passes' stage 1 through the ghost planes of Q)."""
    import threading
    from paper_2505_16992_b200 import linalg, piso, slab
    import test_gpu_slab as T
    dom, c, b = _system((8, 16, 32))
    x_ref, r_ref = _solve(dom, c, b, False, tiled=True, precond=precond)
    u0 = None
    slabs = [slab.SlabDomain(dom, r, world) for r in range(world)]
    slab.SlabComm.local_group(slabs, b.device)
    # the global system restricted to each slab (ghost rows included)
    res = [None] * world
    cs = [sd.scatter(c.t().contiguous()).t().contiguous() for sd in slabs]
    bs = [sd.scatter(b.t().contiguous()).t().contiguous() for sd in slabs]
    torch.cuda.synchronize()
    ready = threading.Barrier(world)

    def work(r):
        s = torch.cuda.Stream(b.device)
        with torch.cuda.stream(s):
            T._prewarm(ready)
            plan = slabs[r].device_plan(b.device)
            res[r] = linalg.bicgstab_solve(plan, cs[r], bs[r], tol=1e-12,
                                           precond=precond)
            s.synchronize()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    x = np.zeros((3, dom.n))
    for sd, (xr, reps) in zip(slabs, res):
        lo = sd.x0 * sd.plane
        x[:, lo:lo + sd.nxl * sd.plane] = xr[:, sd.owned_slice].cpu().numpy()
        assert [q.iterations for q in reps] == [q.iterations for q in r_ref]
    xr = x_ref.cpu().numpy()
    assert np.abs(x - xr).max() / np.abs(xr).max() < 1e-10
