"""Cost of the slab decomposition itself, measured on ONE B200: the C4 step
(forward + FULL adjoint) as `world` slabs in one process (a host thread and
stream each, peers linked through the same peer-memory communicator as the
multi-GPU path) against the undecomposed step.  All slabs share the GPU, so
the slab run's time = the same total work + the decomposition's extra
kernels (halo puts / gets, cross-rank reductions, barriers, the spectral
transposes) + the loss of single-kernel efficiency on 1/world-sized pieces.

    python tools/slab_overhead.py --world 8 --steps 3
"""
import argparse
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("PF_NO_GRAPHS", "1")
os.environ.setdefault("PF_MAX_BATCH", "4")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--shape", default="256,192,256")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2505_16992_b200 import adjoint, channel, mesh, piso, slab
    import test_gpu_slab as T
    shape = tuple(int(v) for v in args.shape.split(","))
    dev = torch.device("cuda:0")
    dom = mesh.make_channel(shape, ratio=1.03)
    u0, nu, _ = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                           seed=0, device=dev)
    dt = 0.3 * (2 * np.pi / shape[0]) / float(u0.abs().max())
    g = torch.Generator(device="cpu").manual_seed(0)
    w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)

    def run(domain, u, wc, forcing, steps, ws):
        st = piso.make_state(domain, u0=u, device=dev)
        its = []
        for _ in range(steps):
            cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(st.u, nu),
                                  tol=1e-8)
            tape = piso.StepTape()
            st, dg = piso.piso_step(domain, st, cfg, ws, tape)
            gr = adjoint.backward_step(domain, tape, adjoint.GradState(
                u=wc, p=torch.zeros(domain.n, dtype=torch.float64,
                                    device=dev)), tol=1e-8)
            its.append((dg.momentum_iterations, dg.pressure_iterations,
                        gr.solve_iterations))
        return its

    # undecomposed
    ws = piso.PisoWorkspace(dom)
    run(dom, u0, w, channel.WallForcing(dom, dev), 2, ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its1 = run(dom, u0, w, channel.WallForcing(dom, dev), args.steps, ws)
    torch.cuda.synchronize()
    t_single = (time.perf_counter() - t0) / args.steps

    slabs = [slab.SlabDomain(dom, r, args.world) for r in range(args.world)]
    comms = slab.SlabComm.local_group(slabs, dev)
    torch.cuda.synchronize()
    ready = threading.Barrier(args.world)
    start = threading.Barrier(args.world)
    out = [None] * args.world
    times = [None] * args.world

    def work(r):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            sd = slabs[r]
            # every allocation of the run is served from this thread's cached
            # block (a cudaMalloc mid-run would wait on the other slabs'
            # spinning kernels): ~1 KB per local cell covers a step + tape
            T._prewarm(ready, nbytes=int(1100 * sd.n))
            ul, wl = sd.scatter(u0), sd.scatter(w).contiguous()
            f = slab.SlabWallForcing(sd, dev)
            wsl = piso.PisoWorkspace(sd)
            s.synchronize()
            start.wait()
            run(sd, ul, wl, f, 2, wsl)
            s.synchronize()
            start.wait()
            t = time.perf_counter()
            out[r] = run(sd, ul, wl, f, args.steps, wsl)
            s.synchronize()
            times[r] = (time.perf_counter() - t) / args.steps
            comms[r].status()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(args.world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    t_slab = max(times)
    print(f"single-domain step {1e3 * t_single:.1f} ms, iterations {its1[-1]}")
    print(f"{args.world} slabs on one GPU: step {1e3 * t_slab:.1f} ms "
          f"(x{t_slab / t_single:.2f}), iterations {out[0][-1]}")
    print(f"decomposition overhead: {100 * (t_slab / t_single - 1):.0f} % "
          f"=> bound on strong-scaling efficiency from extra work alone: "
          f"{100 * t_single / t_slab:.0f} %")


if __name__ == "__main__":
    main()
