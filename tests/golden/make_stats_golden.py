"""Golden vectors of the reference's channel statistics (test fixture).

    python oracle/build_ref.py && python tests/golden/make_stats_golden.py

Runs the reference ``pisoflow.stats`` (S/stats.py) on a small wall-refined
channel: frame profiles of three velocity frames, the cotangent of one frame
profile, the window profile and its backward, the statistics loss with the
turbulent-channel weights and its gradients, and a ChannelAccumulator
profile (means, covariances, skewness, flatness, friction scales).  Writes
tests/golden/stats.npz.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import build_ref  # noqa: E402

build_ref.build()
sys.path.insert(0, build_ref.ref_path())

from pisoflow import mesh, piso, stats  # noqa: E402

SHAPE = (8, 12, 8)
RATIO = 1.1


def main():
    dom = mesh.make_channel(SHAPE, ratio=RATIO)
    rng = np.random.default_rng(7)
    st, nu, u_tau = piso.reichardt_init(dom, 180.0, perturbation=0.1, seed=3)
    frames = [np.asarray(st.u) + 0.05 * k * rng.standard_normal(st.u.shape)
              for k in range(3)]
    sl = stats.channel_slices(dom)
    profiles = [stats.frame_profile(sl, u) for u in frames]
    d_mean = rng.standard_normal(profiles[0][0].shape)
    d_cov = rng.standard_normal(profiles[0][1].shape)
    du = stats.frame_profile_backward(sl, frames[1], d_mean, d_cov)
    wmu, wcov = stats.window_profile(profiles)
    wback = stats.window_profile_backward(profiles, d_mean, d_cov)
    w = stats.tcf_default_weights(3)
    ref = (profiles[0][0] * 0.9, profiles[0][1] * 1.1)
    loss, grads = stats.stats_loss_grad(profiles, ref, w)
    acc = stats.ChannelAccumulator(dom)
    for u in frames:
        acc.add_frame(u, dt=0.1)
    prof = acc.profile(nu=nu)
    out = dict(shape=np.array(SHAPE), ratio=RATIO, nu=nu,
               frames=np.stack(frames), d_mean=d_mean, d_cov=d_cov, du=du,
               y=sl.y, y_lo=sl.y_lo, y_hi=sl.y_hi,
               win_mean=wmu, win_cov=wcov,
               wback_mean=np.stack([m for m, _ in wback]),
               wback_cov=np.stack([c for _, c in wback]),
               ref_mean=ref[0], ref_cov=ref[1], loss=loss,
               grad_mean=np.stack([m for m, _ in grads]),
               grad_cov=np.stack([c for _, c in grads]),
               acc_mean=prof.mean, acc_cov=prof.cov,
               acc_skew=prof.skewness, acc_flat=prof.flatness,
               acc_u_tau=prof.scales.u_tau, acc_time=acc.time)
    for k, (m, c) in enumerate(profiles):
        out[f"mean{k}"] = m
        out[f"cov{k}"] = c
    np.savez(os.path.join(HERE, "stats.npz"), **out)
    print("stats golden: loss", loss, "u_tau", prof.scales.u_tau)


if __name__ == "__main__":
    main()
