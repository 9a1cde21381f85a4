"""Channel statistics (SURVEY.md §8 f) against the reference's own outputs
(tests/golden/stats.npz, made by tests/golden/make_stats_golden.py from
S/stats.py).  CPU tier: slicing and the small-tensor parts (window profile,
its backward, the statistics loss and its gradients).  GPU tier: the frame
moments and their cotangent from libpisob200.so, the streaming accumulator,
the autograd function, and the slab path."""

import os
import threading

import numpy as np
import pytest
import torch

from paper_2505_16992_b200 import mesh, stats

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "stats.npz"))


def _rel(a, b):
    a = a.detach().cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _dom():
    return mesh.make_channel(tuple(int(v) for v in G["shape"]),
                             ratio=float(G["ratio"]))


def _profiles(dev=None):
    return [(torch.as_tensor(G[f"mean{k}"], device=dev),
             torch.as_tensor(G[f"cov{k}"], device=dev)) for k in range(3)]


def test_channel_slices_match_reference():
    sl = stats.channel_slices(_dom())
    assert _rel(sl.y, G["y"]) < 1e-14
    assert sl.y_lo == pytest.approx(float(G["y_lo"]), abs=1e-14)
    assert sl.y_hi == pytest.approx(float(G["y_hi"]), abs=1e-14)
    assert sl.m == 64
    with pytest.raises(ValueError):
        stats.channel_slices(mesh.make_cavity((6, 6)))


def test_window_profile_and_backward_match_reference():
    prof = _profiles()
    mu, cov = stats.window_profile(prof)
    assert _rel(mu, G["win_mean"]) < 1e-13
    assert _rel(cov, G["win_cov"]) < 1e-13
    back = stats.window_profile_backward(prof, G["d_mean"], G["d_cov"])
    for k, (dm, dc) in enumerate(back):
        assert _rel(dm, G["wback_mean"][k]) < 1e-13
        assert _rel(dc, G["wback_cov"][k]) < 1e-13


def test_stats_loss_and_gradients_match_reference():
    prof = _profiles()
    w = stats.tcf_default_weights(3)
    loss, grads = stats.stats_loss_grad(prof, (G["ref_mean"], G["ref_cov"]),
                                        w)
    assert loss == pytest.approx(float(G["loss"]), rel=1e-13)
    for k, (dm, dc) in enumerate(grads):
        assert _rel(dm, G["grad_mean"][k]) < 1e-12
        assert _rel(dc, G["grad_cov"][k]) < 1e-12
    # the differentiable torch form has the same value and gradients
    pr = [(m.clone().requires_grad_(True), c.clone().requires_grad_(True))
          for m, c in prof]
    lt = stats.stats_loss_torch(pr, (G["ref_mean"], G["ref_cov"]), w)
    lt.backward()
    assert float(lt.detach()) == pytest.approx(float(G["loss"]), rel=1e-13)
    for k, (m, c) in enumerate(pr):
        assert _rel(m.grad, G["grad_mean"][k]) < 1e-12
        assert _rel(c.grad, G["grad_cov"][k]) < 1e-12
    with pytest.raises(ValueError):
        stats.LossWeights(mean=[-1.0, 0, 0], cov=np.zeros((3, 3)))


@pytest.mark.gpu
def test_frame_moments_and_backward_on_device():
    dev = torch.device("cuda:0")
    dom = _dom()
    sl = stats.channel_slices(dom)
    for k in range(3):
        u = torch.as_tensor(G["frames"][k], device=dev)
        mean, cov = stats.frame_profile(sl, u)
        assert _rel(mean, G[f"mean{k}"]) < 1e-12
        assert _rel(cov, G[f"cov{k}"]) < 1e-11
    u1 = torch.as_tensor(G["frames"][1], device=dev)
    du = stats.frame_profile_backward(sl, u1, G["d_mean"], G["d_cov"])
    assert _rel(du, G["du"]) < 1e-12
    # autograd: d/du of <d_mean, mean> + <d_cov, cov>
    uu = u1.clone().requires_grad_(True)
    m, c = stats.frame_profile_fn(sl, uu)
    (m * torch.as_tensor(G["d_mean"], device=dev)).sum().add(
        (c * torch.as_tensor(G["d_cov"], device=dev)).sum()).backward()
    assert _rel(uu.grad, G["du"]) < 1e-12


@pytest.mark.gpu
def test_channel_accumulator_on_device():
    dev = torch.device("cuda:0")
    acc = stats.ChannelAccumulator(_dom())
    for k in range(3):
        acc.add_frame(torch.as_tensor(G["frames"][k], device=dev), dt=0.1)
    prof = acc.profile(nu=float(G["nu"]))
    assert _rel(prof.mean, G["acc_mean"]) < 1e-12
    assert _rel(prof.cov, G["acc_cov"]) < 1e-11
    assert _rel(prof.skewness, G["acc_skew"]) < 1e-9
    assert _rel(prof.flatness, G["acc_flat"]) < 1e-9
    assert prof.scales.u_tau == pytest.approx(float(G["acc_u_tau"]),
                                              rel=1e-12)
    assert acc.time == pytest.approx(float(G["acc_time"]))


@pytest.mark.gpu
def test_frame_moments_on_slabs():
    """The slices span the slab ranks (sums added across them)."""
    from paper_2505_16992_b200 import slab
    import test_gpu_slab as T
    dev = torch.device("cuda:0")
    dom = _dom()
    u = torch.as_tensor(G["frames"][2], device=dev)
    slabs = [slab.SlabDomain(dom, r, 2) for r in range(2)]
    slab.SlabComm.local_group(slabs, dev)
    out = [None, None]
    torch.cuda.synchronize()
    ready = threading.Barrier(2)

    def work(r):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            T._prewarm(ready)
            sl = stats.channel_slices(slabs[r])
            out[r] = stats.frame_profile(sl, slabs[r].scatter(u))
            s.synchronize()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    for r in range(2):
        assert _rel(out[r][0], G["mean2"]) < 1e-12
        assert _rel(out[r][1], G["cov2"]) < 1e-11
