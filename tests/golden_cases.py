"""Rebuild the golden-vector cases (tests/golden/make_golden.py) with this
repository's own mesh generators, and load the fixtures."""

import os

import numpy as np

from paper_2505_16992_b200 import mesh

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

ORTHOGONAL = ["cavity8", "box3d", "channel", "twoblock_rot", "backstep",
              "obstacle", "refined_cavity"]
NONORTHO = ["distorted_nonortho", "sheared3d"]
ALL = ORTHOGONAL + NONORTHO


def build(name):
    if name == "cavity8":
        return mesh.make_cavity((8, 8))
    if name == "box3d":
        return mesh.make_box((4, 5, 6))
    if name == "channel":
        return mesh.make_channel((6, 8, 4), ratio=1.1)
    if name == "twoblock_rot":
        return mesh.make_two_block((4, 4), rotated=True)
    if name == "backstep":
        return mesh.make_backstep(cells_per_h=2)
    if name == "obstacle":
        return mesh.make_obstacle_grid(nx=(4, 3, 8), ny=(4, 3, 4))
    if name == "refined_cavity":
        x = mesh.wall_refined_coords(12, 0.5, 1.2)
        blk = mesh.BlockSpec(mesh._grid_vertices(x, x))
        bnd = {(0, a, s): mesh.Dirichlet(0.0) for a in range(2)
               for s in (0, 1)}
        bnd[(0, 1, 1)] = mesh.Dirichlet((1.0, 0.0))
        return mesh.Domain([blk], bnd)
    if name == "distorted_nonortho":
        return mesh.make_poiseuille((6, 4), distort=0.35)
    if name == "sheared3d":
        return sheared3d(mesh)
    raise KeyError(name)


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def split_bc(g, flat):
    off = np.concatenate([[0], np.cumsum(g["bface_m"])]).astype(int)
    return [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def source_of(g):
    s = g["source_given"]
    return None if s.size == 0 else s


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.abs(b).max() if b.size else 0.0, 1e-300)
    return float(np.abs(a - b).max() / scale) if a.size else 0.0


def sheared3d(mesh):
    """Non-orthogonal 3D block: periodic in x and z (faces conformal up to a
    rigid shift), walls at y = 0 / 1 with a moving lid; the walls are not
    plane so their face metrics carry tangential terms."""
    x = np.linspace(0.0, 1.0, 5)
    y = np.linspace(0.0, 1.0, 6)
    z = np.linspace(0.0, 1.0, 5)
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    Xp = X + 0.08 * np.sin(2 * np.pi * Y) * np.cos(2 * np.pi * Z)
    Yp = Y + 0.05 * np.sin(np.pi * Y) * np.cos(2 * np.pi * X)
    Zp = Z + 0.08 * np.sin(2 * np.pi * X) * np.sin(np.pi * Y)
    blk = mesh.BlockSpec(np.stack([Xp, Yp, Zp], axis=-1))
    ident = (0, 1, 2)
    flip = (False, False, False)
    bnd = {(0, 0, 0): mesh.Connection(0, 0, 1, ident, flip),
           (0, 0, 1): mesh.Connection(0, 0, 0, ident, flip),
           (0, 2, 0): mesh.Connection(0, 2, 1, ident, flip),
           (0, 2, 1): mesh.Connection(0, 2, 0, ident, flip),
           (0, 1, 0): mesh.Dirichlet(0.0),
           (0, 1, 1): mesh.Dirichlet((0.5, 0.0, 0.2))}
    return mesh.Domain([blk], bnd)
