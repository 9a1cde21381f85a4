"""CPU tier: channel drivers (initial condition, wall forcing) against the
reference's outputs (tests/golden/reichardt.npz)."""

import numpy as np
import pytest
import torch

import golden_cases as G
from paper_2505_16992_b200 import channel, mesh


@pytest.mark.parametrize("tag", ["a", "b"])
def test_reichardt_box_path_matches_reference(tag):
    g = G.load("reichardt")
    dom = mesh.make_channel(tuple(g[f"{tag}_shape"]),
                            ratio=float(g[f"{tag}_ratio"]))
    u, nu, ut = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=3, device="cpu")
    assert nu == pytest.approx(float(g[f"{tag}_nu"]), rel=1e-15)
    assert ut == pytest.approx(float(g[f"{tag}_utau"]), rel=1e-15)
    assert G.rel(u.numpy(), g[f"{tag}_u"]) < 1e-13
    # the wall forcing is a device kernel: test_gpu_channel.py


def test_reichardt_host_path_matches_reference():
    g = G.load("reichardt")
    dom = mesh.make_channel(tuple(g["a_shape"]), ratio=float(g["a_ratio"]))
    re_cl = (180.0 / 0.116) ** (1.0 / 0.88)
    nu = 1.0 / re_cl
    u = channel._reichardt_host(dom, 180.0, nu, 180.0 * nu, 1.0, 1, 0, 0.1, 3)
    assert G.rel(u, g["a_u"]) < 1e-13
