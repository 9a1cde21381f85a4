"""B200-native differentiable PISO step (arXiv 2505.16992 / PICT path).

Drop-in for the reference ``pisoflow`` hot path: ``mesh`` (Domain and
generators), ``piso`` (piso_step and building blocks), ``adjoint``
(backward_step, backward_rollout, GradientPath, gradcheck), ``linalg``
(cg_solve, bicgstab_solve, SolverError), ``autograd`` (torch.autograd
wrapper) and ``channel`` (turbulent-channel drivers).  All arithmetic runs
in ``libpisob200.so`` (hand-written sm_100a CUDA behind a C ABI); there is no
CPU fallback.
"""

__version__ = "0.1.0"
LANE = "cuda-sm100a"

__all__ = ["mesh", "piso", "adjoint", "linalg", "autograd", "channel",
           "LANE", "__version__"]


def __getattr__(name):
    if name in ("mesh", "piso", "adjoint", "linalg", "autograd", "channel",
                "plan"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
