"""CPU tier: the host side of the slab decomposition (SURVEY.md §8 e).

The partition of the channel into slabs, the slab meshes (metrics, boundary
entries, ghost planes), the global <-> local layouts and, with world_size 2
over gloo, that the ranks' owned cells tile the global mesh exactly.  The
device side (halo exchange, in-kernel reductions, spectral transposes) is
covered by tests/test_gpu_slab*.py on the B200."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_16992_b200 import mesh, slab


@pytest.mark.parametrize("nx,world", [(8, 1), (8, 2), (8, 3), (256, 8),
                                      (7, 4)])
def test_slab_bounds_tile_the_axis(nx, world):
    spans = [slab.slab_bounds(nx, r, world) for r in range(world)]
    x = 0
    for x0, nxl in spans:
        assert x0 == x and nxl >= 1
        x += nxl
    assert x == nx
    assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_slab_mesh_matches_global_mesh(world):
    dom = mesh.make_channel((8, 6, 4), ratio=1.1)
    lx = 2.0 * np.pi
    for r in range(world):
        sd = slab.SlabDomain(dom, r, world)
        assert sd.n == (sd.nxl + 2) * sd.plane
        assert sd.box_layout() == ((sd.nxl + 2, 6, 4), (True, False, True))
        rows = sd._global_rows()
        np.testing.assert_allclose(sd.jac, dom.jac[rows], rtol=1e-14)
        np.testing.assert_allclose(sd.alpha, dom.alpha[rows], rtol=1e-14)
        c, g = sd.centers, dom.centers[rows]
        np.testing.assert_allclose(c[:, 1:], g[:, 1:], rtol=1e-14)
        dx = np.mod(c[:, 0] - g[:, 0] + 0.5 * lx, lx) - 0.5 * lx
        assert np.abs(dx).max() < 1e-12
        # the owned block starts at global plane x0
        own = sd.owned(np.arange(sd.n))
        assert np.array_equal(rows[own], sd.owned_global_rows())


def test_slab_boundary_entries_cover_the_walls():
    dom = mesh.make_channel((8, 6, 4), ratio=1.1)
    world = 3
    got = {(f.axis, f.side): [] for f in dom.bfaces}
    for r in range(world):
        sd = slab.SlabDomain(dom, r, world)
        rows = sd._global_rows()
        lo, hi = sd.plane, sd.plane * (sd.nxl + 1)
        for f in sd.bfaces:
            cells = np.asarray(f.cells)
            owned = cells[(cells >= lo) & (cells < hi)]
            got[(f.axis, f.side)].append(rows[owned])
            # face metrics of the slab entries equal the global ones
            gf = next(x for x in dom.bfaces
                      if (x.axis, x.side) == (f.axis, f.side))
            gidx = {int(c): k for k, c in enumerate(gf.cells)}
            k = [gidx[int(rows[c])] for c in cells]
            np.testing.assert_allclose(f.face_jac, gf.face_jac[k], rtol=1e-14)
            np.testing.assert_allclose(f.face_alpha, gf.face_alpha[k],
                                       rtol=1e-14)
    for f in dom.bfaces:
        allc = np.sort(np.concatenate(got[(f.axis, f.side)]))
        assert np.array_equal(allc, np.sort(np.asarray(f.cells)))


def test_scatter_gather_and_boundary_values_roundtrip():
    dom = mesh.make_channel((8, 6, 4), ratio=1.1)
    rng = np.random.default_rng(0)
    u = rng.standard_normal((dom.n, 3))
    bc = [rng.standard_normal((f.m, 3)) for f in dom.bfaces]
    out = np.zeros_like(u)
    for r in range(4):
        sd = slab.SlabDomain(dom, r, 4)
        loc = sd.scatter(u)
        assert loc.shape == (sd.n, 3)
        np.testing.assert_array_equal(loc, u[sd._global_rows()])
        sd.gather_into(loc, out)
        tl = sd.scatter(torch.as_tensor(u))
        assert torch.equal(tl, torch.as_tensor(loc))
        lbc = sd.local_bc(bc)
        for f, v in zip(sd.bfaces, lbc):
            gf = next(x for x in dom.bfaces
                      if (x.axis, x.side) == (f.axis, f.side))
            gv = bc[dom.bfaces.index(gf)]
            gidx = {int(c): k for k, c in enumerate(gf.cells)}
            rows = sd._global_rows()
            k = [gidx[int(rows[c])] for c in f.cells]
            np.testing.assert_array_equal(v, gv[k])
    np.testing.assert_array_equal(out, u)


def test_slab_rejects_unsupported_domains():
    with pytest.raises(ValueError):
        slab.SlabDomain(mesh.make_cavity((8, 8)), 0, 2)       # walls on x
    with pytest.raises(ValueError):
        slab.SlabDomain(mesh.make_channel((2, 6, 4)), 0, 4)   # empty slab
    with pytest.raises(ValueError):
        slab.SlabDomain(mesh.make_backstep(2), 0, 2)          # multi-block


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dom = mesh.make_channel((8, 6, 4), ratio=1.1)
    sd = slab.SlabDomain(dom, rank, world)
    mine = torch.as_tensor(sd.owned_global_rows())
    sizes = [None] * world
    dist.all_gather_object(sizes, int(mine.numel()))
    parts = [torch.empty(s, dtype=mine.dtype) for s in sizes]
    dist.all_gather(parts, mine)
    # wall-cell counts per wall: local owned counts summed over the ranks
    lo, hi = sd.plane, sd.plane * (sd.nxl + 1)
    counts = torch.tensor([float(((np.asarray(f.cells) >= lo)
                                  & (np.asarray(f.cells) < hi)).sum())
                           for f in sd.bfaces], dtype=torch.float64)
    dist.all_reduce(counts)
    if rank == 0:
        torch.save({"rows": torch.cat(parts), "counts": counts}, out)
    dist.barrier()
    dist.destroy_process_group()


def test_owned_cells_tile_the_mesh_world2(tmp_path):
    out = str(tmp_path / "slab.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = torch.load(out)
    dom = mesh.make_channel((8, 6, 4), ratio=1.1)
    assert torch.equal(res["rows"], torch.arange(dom.n))
    assert res["counts"].tolist() == [float(f.m) for f in dom.bfaces]


def test_auto_momentum_preconditioner_per_plan(monkeypatch):
    """precond="ilu0" resolves to Neumann-2 on one domain and to Jacobi on a
    slab plan of several ranks (measured cheaper there); a one-rank slab
    keeps Neumann-2; PF_MOMENTUM_PRECOND (read at import) overrides both."""
    from types import SimpleNamespace
    from paper_2505_16992_b200 import linalg
    dom = mesh.make_channel((8, 16, 32), ratio=1.05)
    plans = {w: SimpleNamespace(domain=slab.SlabDomain(dom, 0, w))
             for w in (1, 2, 8)}
    single = SimpleNamespace(domain=dom)
    monkeypatch.setattr(linalg, "_DEFAULT_MOM_PRECOND", "neumann2")
    monkeypatch.setattr(linalg, "_SLAB_MOM_PRECOND", "jacobi")
    assert linalg.auto_momentum_precond(single) == linalg.PRECOND_NEUMANN2
    assert linalg.auto_momentum_precond(plans[1]) == linalg.PRECOND_NEUMANN2
    for w in (2, 8):
        assert linalg.auto_momentum_precond(plans[w]) == linalg.PRECOND_JACOBI
    monkeypatch.setattr(linalg, "_SLAB_MOM_PRECOND", "neumann2")
    assert linalg.auto_momentum_precond(plans[8]) == linalg.PRECOND_NEUMANN2
    monkeypatch.setattr(linalg, "_DEFAULT_MOM_PRECOND", "jacobi")
    assert linalg.auto_momentum_precond(single) == linalg.PRECOND_JACOBI
