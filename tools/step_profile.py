"""Run W warm-up fwd+adjoint steps of a bench config, then ONE step inside
cudaProfilerStart/Stop, so `ncu --profile-from-start off` captures exactly
the kernels of one step.  Developer tool (profiles/), not the bench.

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file out.csv \
        python tools/step_profile.py --config c4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2505_16992_b200 import adjoint, piso
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    bargs = argparse.Namespace(config=args.config)
    dom, state, nu, dt, forcing, w, _ = bench.build_workload(bargs, dev)
    cot = adjoint.GradState(u=w, p=torch.zeros(dom.n, dtype=torch.float64,
                                               device=dev))
    ws = piso.PisoWorkspace(dom)

    def step(state):
        cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(state.u, nu),
                              tol=args.tol)
        tape = piso.StepTape()
        new, dg = piso.piso_step(dom, state, cfg, ws, tape)
        g = adjoint.backward_step(dom, tape, cot, tol=args.tol)
        return new, dg, g

    for _ in range(args.warmup):
        state, _, _ = step(state)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.cudart().cudaProfilerStart()
    e0.record()
    state, dg, g = step(state)
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"step ms {e0.elapsed_time(e1):.3f} mom_it {dg.momentum_iterations} "
          f"p_it {dg.pressure_iterations} adj_it {g.solve_iterations}")


if __name__ == "__main__":
    main()
