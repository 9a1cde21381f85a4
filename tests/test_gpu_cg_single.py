"""GPU tier: the Chronopoulos-Gear pressure CG -- one fused reduction per
iteration ("single"), or two with the residual test in the update pass
("split", the slab plans' default) -- against the
classic three-reduction loop on the same systems (multigrid and spectral
preconditioners, cold and warm starts, zero right-hand side, maxiter 1),
with the production CUDA graphs on and off, and against the exact solve.
The variant is fixed per process (PF_CG_VARIANT), so each runs in a child
(tests/cg_variant_child.py)."""

import os
import subprocess
import sys

import numpy as np
import pytest

import golden_cases as G
from oracle import pisoref as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, variant, graphs):
    out = str(tmp_path / f"{variant}_{int(graphs)}.npz")
    env = dict(os.environ, PF_CG_VARIANT=variant,
               PF_NO_GRAPHS="0" if graphs else "1")
    env.pop("PF_MAX_BATCH", None)  # production batching
    subprocess.run([sys.executable, os.path.join(HERE, "cg_variant_child.py"),
                    out], check=True, env=env, timeout=600)
    return np.load(out)


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    t = tmp_path_factory.mktemp("cgvar")
    return {k: _run(t, *k) for k in VARIANTS}


VARIANTS = [("classic", True), ("single", True), ("single", False),
            ("split", True), ("split", False)]


def test_single_reduction_matches_classic(runs):
    import cg_variant_child as C
    ref = runs[("classic", True)]
    worst = {}
    for key in ref.files:
        if not key.endswith("_rep"):
            continue
        base = key[:-4]
        rc = ref[key]
        for k in VARIANTS[1:]:
            rs = runs[k][key]
            # cold solve and warm-started solve: both converge, iteration
            # counts within one (round-off at the threshold)
            assert rs[1] == 1 and rs[4] == 1, (k, base, rs)
            assert abs(rs[0] - rc[0]) <= 1 and abs(rs[3] - rc[3]) <= 1, \
                (k, base, rs, rc)
            tol = float(base.rsplit("_", 1)[1])
            for sfx in ("_x", "_x2"):
                e = G.rel(runs[k][base + sfx], ref[base + sfx])
                worst[(k, base + sfx)] = e
                assert e < 1e3 * tol, (k, base + sfx, e)
                assert abs(runs[k][base + sfx].mean()) < 1e-12
    # graphs on / off: the same kernels in the same order, bitwise
    for v in ("single", "split"):
        for key in runs[(v, True)].files:
            assert np.array_equal(runs[(v, True)][key],
                                  runs[(v, False)][key]), (v, key)
        for name in C.domains():
            z = runs[(v, True)][name + "_zero"]
            assert z[0] == 0 and z[1] == 1 and z[2] == 0.0
            m1 = runs[(v, True)][name + "_max1"]
            assert m1[0] == ref[name + "_max1"][0]
    print("\n[single-reduction CG] worst rel. diff vs classic: "
          + f"{max(worst.values()):.1e}")


def test_single_reduction_matches_exact(runs):
    import cg_variant_child as C
    from paper_2505_16992_b200 import mesh  # noqa: F401
    for name, (build, _) in C.domains().items():
        dom = build()
        if dom.n > 20000:
            continue
        K = C.pressure_operator(dom)
        b = np.random.default_rng(7).standard_normal(dom.n)
        ex = O.solve_pressure_exact(dom, K, b)
        for v in ("single", "split"):
            x = runs[(v, True)][f"{name}_1e-11_x"]
            assert G.rel(x, ex) < 1e-8, (v, name, G.rel(x, ex))
