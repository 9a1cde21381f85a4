"""Benchmark: forward + adjoint PISO steps on the 3D turbulent channel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5|c5train|slab8] [--no-cpu-baseline]

--gpus N > 1 without torchrun starts the N ranks itself.

Metric (BASELINE.json): Mcell-steps/s of forward+adjoint PISO on the 3D
channel; one "step" = one taped ``piso_step`` plus its ``backward_step``
(FULL gradient path) for a fixed cotangent, on the C4 workload
make_channel((256, 192, 256), ratio=1.03) + reichardt_init(Re_tau=180,
perturbation 0.1, seed 0), dt = 0.3 (2 pi/256) / max|u0|, tol 1e-8, fp64,
per-step wall forcing.  The state advances, warm starts are on (the
reference's run_rollout setting), inputs (>10 GB working set) exceed L2.

Multi-GPU (torchrun, N>1): C4 is slab-decomposed along its periodic
streamwise axis, one slab per rank (strong scaling: the job advances the
one 256x192x256 channel); ghost planes, solver reductions and the spectral
preconditioner's transposes move over NVLink peer memory (paper_2505_16992_
b200/slab.py).  value = global cells x steps / max-over-ranks device time.
The other configs run one replica per rank (weak scaling).

--impl reference runs the reference's own CPU implementation (pisoflow,
built unmodified into oracle/_ref by oracle/build_ref.py) on rank 0, one
single-threaded process per host core, each advancing a bounded
sample of the workload (the same channel recipe at 64x48x64 cells).
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# load every kernel at context creation: a lazy load is a context-wide
# synchronisation, which the spinning cross-rank waits of the slab path
# must not meet mid-run (and it keeps first-launch costs out of warm-up)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

METRIC = "Mcell-steps/s fwd+adjoint PISO, 3D channel"
UNIT = "Mcell-steps/s"

CONFIGS = {
    # name: (shape, ratio, cfl factor, description)
    "c4": ((256, 192, 256), 1.03, 0.3,
           "C4 channel 256x192x256 Re_tau=180, fwd+adjoint"),
    "c5": ((64, 48, 64), 1.095, 0.5,
           "C5 channel 64x48x64 Re_tau=180 (per sample), fwd+adjoint"),
    "slab8": ((128, 96, 128), 1.03, 0.3,
              "C4 per-GPU slab proxy 128x96x128, fwd+adjoint"),
    "c5train": ((64, 48, 64), 1.095, 0.5,
                "C5 LES training step: 64x48x64 sample per GPU, learned SGS "
                "CNN corrector, 16-step unrolled fwd+adjoint, statistics "
                "loss, data parallel"),
}
UNROLL = 16
SAMPLE_SHAPE = (64, 48, 64)

# 2D BASELINE configs (BASELINE.md §3a recipes): name -> description, tol.
# One step = one taped piso_step + its FULL backward_step, as for C4.
CASES2D = {
    "c1": ("C1 lid-driven cavity 32x32 Re=100 (nu 0.01, dt 0.02), "
           "fwd+adjoint", 1e-10),
    "c2": ("C2 lid-driven cavity 1024x1024 wall-refined (ratio 1.0045) "
           "Re=1000 (nu 1e-3, dt 25 dx_min), fwd+adjoint", 1e-8),
    "c3": ("C3 obstacle (Karman) grid 2048x512 in 8 blocks, Re=100 "
           "(inflow 1, nu 0.01, dt 0.0125), fwd+adjoint", 1e-8),
}


def case_2d(mesh, name, sample=False):
    """Domain, nu, dt and initial velocity (n, 2) of a 2D config, built
    with `mesh` -- ours or the reference's (same API: S/mesh.py:476-700).
    `sample`: the same recipe at 1/16 of the cells (the bounded CPU
    baseline of C2 / C3)."""
    import numpy as np
    if name == "c1":
        dom = mesh.make_cavity((32, 32))
        return dom, 0.01, 0.02, np.zeros((dom.n, 2))
    if name == "c2":
        m = 256 if sample else 1024
        x = mesh.wall_refined_coords(m, 0.5, 1.0045)
        blk = mesh.BlockSpec(mesh._grid_vertices(x, x))
        bnd = {(0, a, s_): mesh.Dirichlet(0.0) for a in range(2)
               for s_ in (0, 1)}
        bnd[(0, 1, 1)] = mesh.Dirichlet((1.0, 0.0))
        dom = mesh.Domain([blk], bnd)
        return dom, 1e-3, 25.0 * float(np.diff(x).min()), np.zeros((dom.n, 2))
    if name == "c3":
        f = 4 if sample else 1

        def inlet(fc):
            return np.stack([np.ones(len(fc)), np.zeros(len(fc))], axis=-1)
        dom = mesh.make_obstacle_grid(
            domain_size=(32.0, 8.0), obstacle_center=(6.5, 4.0),
            obstacle_size=(1.0, 1.0),
            nx=(384 // f, 64 // f, 1600 // f), ny=(224 // f, 64 // f, 224 // f),
            inlet=inlet)
        u0 = np.zeros((dom.n, 2))
        u0[:, 0] = 1.0
        return dom, 0.01, 0.0125 * f, u0
    raise KeyError(name)
CPU_SAMPLE_STEPS = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4",
                    choices=sorted(CONFIGS) + sorted(CASES2D))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=20)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--reference-worker", action="store_true",
                    help=argparse.SUPPRESS)
    ap.add_argument("--worker-steps", type=int, default=1,
                    help=argparse.SUPPRESS)
    ap.add_argument("--worker-shape", default="64,48,64",
                    help=argparse.SUPPRESS)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# reference CPU arm


def reference_worker(args):
    """One single-threaded reference process: build the channel with the
    reference's own API (make_channel + reichardt_init + wall forcing, the
    C4 recipe at `--worker-shape`), take `worker-steps` taped fwd+adjoint
    steps, print one JSON progress line per phase (domain build and initial
    condition excluded from the timing)."""
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
              "PISOFLOW_THREADS"):
        os.environ[k] = "1"
    from oracle import build_ref
    sys.path.insert(0, build_ref.ref_path())
    import numpy as np
    from pisoflow import adjoint, kernels, mesh, piso
    tb = time.perf_counter()
    if args.config in CASES2D:
        dom, nu, dt, u0 = case_2d(mesh, args.config,
                                  sample=args.worker_shape == "sample")
        state = piso.make_state(dom, u0=u0)
        shape = (args.worker_shape,)

        def source(u):
            return None
    else:
        shape = tuple(int(v) for v in args.worker_shape.split(","))
        _, ratio, cfl, _ = CONFIGS[args.config]
        dom = mesh.make_channel(shape, ratio=ratio)
        state, nu, u_tau = piso.reichardt_init(dom, 180.0, perturbation=0.1,
                                               seed=0)
        dt = cfl * (2 * np.pi / shape[0]) / np.abs(state.u).max()

        def source(u):
            return piso.wall_forcing_source(dom, u, nu)
    rng = np.random.default_rng(0)
    w = rng.standard_normal((dom.n, dom.dim))
    ws = piso.PisoWorkspace(dom)

    def emit(**kw):
        print(json.dumps(kw), flush=True)

    emit(phase="setup", seconds=time.perf_counter() - tb, n=dom.n)
    t0 = time.perf_counter()
    iters, fwd_s, bwd_s = [], 0.0, 0.0
    for k in range(args.worker_steps):
        ta = time.perf_counter()
        cfg = piso.StepConfig(dt=dt, nu=nu, source=source(state.u),
                              tol=args.tol)
        tape = piso.StepTape()
        state, dg = piso.piso_step(dom, state, cfg, ws, tape)
        tf = time.perf_counter()
        emit(phase="forward", step=k, seconds=tf - ta,
             iterations=[dg.momentum_iterations, dg.pressure_iterations])
        g = adjoint.backward_step(dom, tape,
                                  adjoint.GradState(u=w, p=np.zeros(dom.n)),
                                  tol=args.tol)
        tg = time.perf_counter()
        emit(phase="backward", step=k, seconds=tg - tf,
             iterations=g.solve_iterations)
        fwd_s += tf - ta
        bwd_s += tg - tf
        iters.append((dg.momentum_iterations, dg.pressure_iterations,
                      g.solve_iterations))
    sec = time.perf_counter() - t0
    emit(phase="done", cell_steps=dom.n * args.worker_steps, seconds=sec,
         forward_seconds=fwd_s, backward_seconds=bwd_s, lane=kernels.LANE,
         iterations=iters, shape=list(shape))


def _worker_cmd(shape, steps, tol, config="c4"):
    return [sys.executable, os.path.abspath(__file__), "--reference-worker",
            "--config", config, "--worker-shape", ",".join(map(str, shape)),
            "--worker-steps", str(steps), "--tol", str(tol)]


def run_reference_sample(procs, steps, tol, shape=None, config="c4"):
    """Run `procs` concurrent reference workers; aggregate Mcell-steps/s."""
    cmd = _worker_cmd(shape or SAMPLE_SHAPE, steps, tol, config)
    t0 = time.perf_counter()
    ps = [subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                           text=True, cwd=ROOT) for _ in range(procs)]
    outs = []
    for p in ps:
        o, e = p.communicate(timeout=1800)
        if p.returncode != 0:
            raise RuntimeError(f"reference worker failed: {e[-2000:]}")
        outs.append(json.loads(o.strip().splitlines()[-1]))
    wall = time.perf_counter() - t0
    cells = sum(o["cell_steps"] for o in outs)
    slowest = max(o["seconds"] for o in outs)
    return {"value": cells / slowest / 1e6, "seconds": slowest,
            "cell_steps": cells, "procs": procs, "lane": outs[0]["lane"],
            "iterations": outs[0]["iterations"], "wall": wall}


def run_reference_full(shape, steps, tol, budget_s, config="c4"):
    """The reference on the full workload in ONE single-threaded process
    (the reference is serial: S/_kernels_c.pyx loops, NumPy elementwise).
    Returns the worker's phase records; a run that would overrun `budget_s`
    is stopped and reported as such (never extrapolated)."""
    p = subprocess.Popen(_worker_cmd(shape, steps, tol, config),
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                         text=True, cwd=ROOT)
    recs = []
    timer = threading.Timer(budget_s, p.kill)
    timer.start()
    try:
        for line in p.stdout:
            line = line.strip()
            if line.startswith("{"):
                recs.append(json.loads(line))
        p.wait()
    finally:
        timer.cancel()
    err = p.stderr.read()
    if p.returncode != 0:
        raise RuntimeError(
            f"reference C4 run stopped (rc {p.returncode}) after phases "
            f"{[r.get('phase') for r in recs]}: {err[-500:]}")
    return recs


def reference_arm(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, built
    unmodified) on the SAME workload and config as our arm.  The reference
    is single-threaded, so the C4 step runs in one process on one core; a
    C4 fwd+adjoint step takes ~20 min there, so the arm times
    `PF_REF_STEPS` (default 1) steps regardless of --steps and says so
    (no warm-up: domain construction and the initial condition are outside
    the timed region, and every reference solve is cold-started the same
    way as the first timed step of a warm run).  A bounded 64x48x64 sample
    on all host cores (one process each) is reported beside it, labelled."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                else (os.cpu_count() or 1))
    is2d = args.config in CASES2D
    if is2d:
        args.tol = CASES2D[args.config][1]
    shape = ("full",) if is2d else CONFIGS[args.config][0]
    # C1 is small: all requested steps; the others one step (BASELINE.md
    # §2: C2-C4 one taped step fwd + backward on one core)
    steps = args.steps if args.config == "c1" else \
        int(os.environ.get("PF_REF_STEPS", "1"))
    budget = float(os.environ.get("PF_REF_BUDGET_S", "1650"))
    try:
        from oracle import build_ref
        if not build_ref.build():
            raise RuntimeError("oracle/_ref missing")
        t0 = time.perf_counter()
        sample = None if is2d else run_reference_sample(procs, 1, args.tol)
        recs = run_reference_full(shape, steps, args.tol,
                                  budget - (time.perf_counter() - t0),
                                  args.config)
    except Exception as exc:  # the oracle always exists; report why not
        print(json.dumps({"impl": "reference", "unavailable": str(exc)[:300]}))
        return
    done = recs[-1]
    setup = recs[0]
    value = done["cell_steps"] / done["seconds"] / 1e6
    desc = (f"reference pisoflow (lane {done['lane']}), the full "
            f"{'x'.join(map(str, shape))} workload, {steps} taped fwd+FULL "
            f"adjoint step(s) in one single-threaded process (the reference "
            f"is serial); domain build + initial condition "
            f"{setup['seconds']:.0f} s excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": UNIT, "n_gpus": args.gpus, "steps": steps, "warmup": 0,
        "requested": {"steps": args.steps, "warmup": args.warmup},
        "ms_per_step": 1e3 * done["seconds"] / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1,
                         "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_seconds": {"forward": done["forward_seconds"],
                              "backward": done["backward_seconds"],
                              "setup": setup["seconds"]},
        "reference_iterations": done["iterations"],
    }
    if sample is not None:
        line["all_cores_sample"] = {
            "value": sample["value"], "unit": UNIT, "cores": procs,
            "what": (f"NOT the same config: {procs} concurrent single-"
                     f"threaded reference processes, each 1 fwd+adjoint "
                     f"step of the channel recipe at "
                     f"{'x'.join(map(str, SAMPLE_SHAPE))}"),
            "iterations": sample["iterations"]}
    print(json.dumps(line))


def workload_config(args):
    if args.config in CASES2D:
        desc, tol = CASES2D[args.config]
        return {"workload": desc, "tol": tol, "gradient_path": "full",
                "parallelism": "single" if args.gpus <= 1 else "replicas",
                "l2": ("C1 fits in L2 (latency-bound, no flush)"
                       if args.config == "c1" else
                       "inputs larger than L2 (no flush needed)")}
    shape, ratio, cfl, desc = CONFIGS[args.config]
    return {"workload": desc, "grid": list(shape),
            "cells": int(math.prod(shape)), "wall_ratio": ratio,
            "dt_rule": f"{cfl}*(2pi/{shape[0]})/max|u0|", "tol": args.tol,
            "gradient_path": "full",
            "parallelism": (("single" if args.gpus <= 1 else
                             f"slab{args.gpus} (x split, NVLink P2P halos)"
                             if args.config in ("c4", "slab8") else
                             "replicas")),
            "l2": "inputs larger than L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# clocks


def wait_for_idle_gpu(index, timeout_s=60.0):
    """Other processes on this GPU (e.g. a test run's stragglers) would share
    its SMs and HBM during the timed region: wait up to timeout_s for them
    to leave.  Returns the PIDs still there (reported on the line)."""
    if os.environ.get("PF_NO_IDLE_WAIT") == "1":  # diagnosis only
        return []
    me = os.getpid()
    t0 = time.time()
    others = []
    while True:
        try:
            out = subprocess.run(
                ["nvidia-smi", "--query-compute-apps=pid", "--format=csv,noheader",
                 "-i", str(index)], capture_output=True, text=True,
                timeout=10).stdout
            others = [int(x) for x in out.split() if x.strip().isdigit()
                      and int(x) != me]
        except (OSError, subprocess.SubprocessError, ValueError):
            return []
        if not others or time.time() - t0 > timeout_s:
            return others
        time.sleep(1.0)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 250 ms by a reader
    thread.  start() returns once the first sample has arrived, so the
    sampler's own start-up (which touches the GPU) is outside the timed
    region; stop() keeps only the samples taken while the region ran."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,"
             "clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t_start = None
        self.first = threading.Event()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line))
            self.first.set()

    def start(self):
        if os.environ.get("PF_NO_CLOCK_SAMPLER") == "1":  # diagnosis only
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("PF_CLOCK_MS", "250")],
                stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()
        self.first.wait(timeout=10)

    def mark(self):
        """Start of the timed region."""
        self.t_start = time.perf_counter()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        t_end = time.perf_counter()
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        t0 = self.t_start if self.t_start is not None else 0.0
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for t, line in list(self.lines):
            if t < t0 or t > t_end + 0.2:
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm


# algorithmic bytes per cell (3D fp64) of the pressure-solver kernels, as
# tabulated in DESIGN.md: minimum traffic with every array read or written
# once and stencil neighbours reused on chip
KERNEL_BYTES = {
    "k_cg_spmv_faces": 40,        # 3 face weights + p + q
    "k_cg_spmv": 40,              # survey SpMV_P minimum (stencil form moves 72)
    "k_cg_spmv_pt": 56,           # tiled: z, p, 3 faces in; p', q out
    "k_cg_update": 48,            # x, p, r, q read; x, r written
    # damped block-Jacobi Y-line smoother (Thomas factors precomputed)
    "k_mg_smooth0 (level 0)": 40,         # r, 1/den, w_y, c' read; x written
    "k_mg_resid_restrict (level 0)": 41,  # r, x, 3 faces; 1/8 coarse r
    "k_mg_prolong_resid (level 0)": 49,   # r, x, 3 faces, 1/8 coarse x; res
    # final pass with the CG z-sums fused: res, 1/den, w_y, c', r, x r+w,
    # 1/8 coarse x
    "k_mg_smooth2_cg (level 0)": 57,
    "k_cg_pupdate": 24,           # z, p read; p written
    # spectral preconditioner: the (Y, kz, kx) work array holds ~n/2
    # complex values, 8 B per cell per sweep
    "k_spec_fwd_z": 16,           # r read; spectrum written
    "k_spec_x (forward)": 16,     # spectrum read + written
    "k_spec_ysolve": 16,          # minimum: spectrum read + written once
    "k_spec_x (inverse)": 16,
    "k_spec_inv_z + CG z-sums": 24,  # spectrum, r read; z written
}

# batched BiCGStab (3 components sharing the 7-row stencil C, Jacobi):
# pv: C rows 56 + per comp r, p, v, rhat read, p', v' written (48)
# st: C rows 56 + per comp r, v read, t written (24)
# xr: diag 8 + per comp x r/w, p, r, v, t, rhat read, r written (64)
BI_BYTES = {"k_bi_pv": 56 + 3 * 48, "k_bi_st": 56 + 3 * 24,
            "k_bi_xr": 8 + 3 * 64,
            # Neumann-2 passes (kernel_bytes): 6 off-diagonal rows + 1/A
            "k_bi_nm_rpv": 48 + 8 + 3 * 80, "k_bi_nm_st": 48 + 8 + 3 * 32}


def kernel_bytes(nm, d):
    """Algorithmic bytes per cell of kernel `nm` in d dimensions (the
    tables above are the 3D figures; stencils carry 2d+1 rows, the face
    form d faces, the multigrid transfers 1/2^d coarse values)."""
    rows = 2 * d + 1
    bi = {"k_bi_pv": 8 * rows + d * 48, "k_bi_st": 8 * rows + d * 24,
          "k_bi_xr": 8 + d * 64,
          # Neumann-2: 2d off-diagonal rows + 1/A; per component the merged
          # pass reads r, v, p, t, r^, z and writes r', z, p', v'; st reads
          # r, v', r^ and writes t
          "k_bi_nm_rpv": 16 * d + 8 + d * 80,
          "k_bi_nm_st": 16 * d + 8 + d * 32}
    if nm in bi:
        return bi[nm]
    co = 8.0 / 2 ** d
    dep = {"k_cg_spmv_faces": 8 * (d + 2),
           # tiled direction update + SpMV: z, p, d faces in; p', q out
           "k_cg_spmv_pt": 8 * (d + 2) + 16,
           # stencil form (Jacobi plans: multi-block grids): rows + p + q
           "k_cg_spmv": 8 * rows + 16,
           "k_mg_resid_restrict (level 0)": 8 * (2 + d) + co,
           "k_mg_prolong_resid (level 0)": 8 * (3 + d) + co,
           "k_mg_smooth2_cg (level 0)": 56 + co}
    return dep.get(nm, KERNEL_BYTES.get(nm))


MG_NAMES = ["k_mg_smooth0 (level 0)", "k_mg_resid_restrict (level 0)",
            "mg coarse levels", "k_mg_prolong_resid (level 0)",
            "k_mg_smooth2_cg (level 0)", "zsum (fused into smooth2)"]
SPEC_NAMES = ["k_spec_fwd_z", "k_spec_x (forward)", "k_spec_ysolve",
              "k_spec_x (inverse)", "k_spec_inv_z + CG z-sums",
              "zsum (fused into inv_z)"]


def _lockstep(reports, prefix, d):
    """Lock-step iterations of the batched BiCGStab solves whose stage
    label starts with `prefix` (the d components of one solve run
    together, so a solve costs max over its components)."""
    its = [r.iterations for r in reports if r.stage.startswith(prefix)]
    return sum(max(its[k:k + d]) for k in range(0, len(its), d))


def measure_roofline(args, dom, plan, state, nu, dt, dev, per_step):
    """Live per-kernel timing (CUDA events on the launching stream) of the
    two solver iterations that make up most of the step -- the batched
    BiCGStab of the momentum predictor and its adjoint (pf_bicgstab_profile)
    and the preconditioned pressure CG (pf_cg_profile) -- on this step's
    operators.  Each kernel's share of the step is its per-launch time x
    launches per step (from the step's own iteration counts) / step time;
    the roofline entry is the kernel with the largest share."""
    import ctypes
    import torch
    from paper_2505_16992_b200 import _lib
    from paper_2505_16992_b200 import piso as P
    c = P.assemble_momentum(dom, state.u, nu, dt)
    k = torch.empty_like(c)
    _lib.call("pf_assemble_pressure", plan.handle, _lib.ptr(c), 0,
              _lib.ptr(k), plan.stream)
    b = torch.randn(dom.n, dtype=torch.float64, device=dev)
    mg = plan.has_mg
    if mg:
        plan.mg_prepare(k)
    ms = (ctypes.c_double * 12)()
    _lib.call("pf_cg_profile", plan.handle, _lib.ptr(k), _lib.ptr(b),
              args.profile_iters, 2 if mg else 1, _lib.ptr(plan.workspace),
              _lib.ptr(plan.mg_workspace if mg else None), ms, plan.stream)
    cgt = ms[11] == 1.0   # the direction update rides in the tiled SpMV
    names = (["k_cg_spmv_pt" if cgt else
              "k_cg_spmv_faces" if mg else "k_cg_spmv", "k_cg_update"]
             + ((SPEC_NAMES if plan.geom_kind == "spectral" else MG_NAMES)
                if mg else [None] * 6) + [None if cgt else "k_cg_pupdate"])
    cg = {}
    for j, nm in enumerate(names):
        if nm is not None and nm in KERNEL_BYTES and ms[j] > 0:
            cg[nm] = float(ms[j])
    d = dom.dim
    bb = torch.randn((d, dom.n), dtype=torch.float64, device=dev)
    bi = {}
    for trans, tag in ((0, ""), (1, " (adjoint)")):
        bm = (ctypes.c_double * 5)()
        _lib.call("pf_bicgstab_profile", plan.handle, _lib.ptr(c), trans, d,
                  _lib.ptr(bb), 8, _lib.ptr(plan.workspace), bm, plan.stream)
        # Neumann-2: the x/r update rides in the next pv pass (k_bi_nm_rpv)
        names = (("k_bi_nm_rpv", "k_bi_nm_st", None) if bm[4] == 3
                 else ("k_bi_pv", "k_bi_st", "k_bi_xr"))
        for j, nm in enumerate(names):
            if nm is not None:
                bi[nm + tag] = float(bm[j])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # cells one launch processes: the owned cells (a slab's ghost planes are
    # only read)
    n = dom.nxl * dom.plane if hasattr(dom, "nxl") else dom.n
    launches = {}
    for nm in bi:
        launches[nm] = per_step["bi_adj" if "adjoint" in nm else "bi_fwd"]
    for nm in cg:
        launches[nm] = per_step["cg"]
    allk = dict(cg)
    allk.update(bi)

    def nbytes(nm):
        return kernel_bytes(nm.replace(" (adjoint)", ""), d)

    share = {nm: allk[nm] * launches[nm] / per_step["ms"] for nm in allk}
    top = max(share, key=share.get)
    gbs = {nm: nbytes(nm) * n / (allk[nm] * 1e-3) / 1e9 for nm in allk}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(top)
        except (OSError, ValueError, AttributeError):
            traffic = None
    it_ms = float(ms[9])
    return {"bound": "hbm", "kernel": top, "achieved": gbs[top], "peak": peak,
            "unit": "GB/s", "frac": gbs[top] / peak, "traffic": traffic,
            "peak_source": peak_src, "bytes_per_cell": nbytes(top),
            "cells_per_launch": n, "ms_per_launch": allk[top],
            "share_of_step": share[top],
            "kernels": {nm: {"ms_per_launch": allk[nm],
                             "launches_per_step": launches[nm],
                             "share_of_step": share[nm],
                             "bytes_per_cell": nbytes(nm),
                             "achieved_gbs": gbs[nm],
                             "frac": gbs[nm] / peak}
                        for nm in sorted(allk, key=lambda x: -share[x])},
            "pressure_cg_iteration": {
                "preconditioner": plan.geom_kind if mg else "jacobi",
                "ms": it_ms, "ms_graph_replay": float(ms[10])},
            "whole_step": whole_step_bytes(d, per_step, n, peak,
                                           nm_bi="k_bi_nm_rpv" in "".join(bi))}


def whole_step_bytes(d, per_step, n, peak, nm_bi):
    """SURVEY.md §8(d)'s whole-step figure: sum over the step's kernels of
    algorithmic bytes/cell x invocations (from the step's own iteration
    counts), times the cells, over the measured step time.  Per-op bytes
    (fp64, s = 8, q = 2d+1 stencil rows):
      momentum assembly + rhs 16 s; pressure assembly (2d+2) s;
      BiCGStab per lock-step iteration: this repo's passes (Neumann-2: the
        merged x/r + pv pass and st, 448 B; Jacobi: pv, st, x/r, 528 B in
        3D) + per solve the init pass (reads b, x,
        C; writes r, r^, 1/A), the verification (b, x, C) and, Neumann-2,
        the close pass (z, 1/A, N, x);
      per corrector: h-stage + divergence (q+3d+1) s, correction (2d+2) s;
      CG per iteration: SpMV_P (d+2) s + update 6 s + preconditioner
        (spectral: 11 s, 4 Fourier / line sweeps over the n/2-complex
        spectrum) + direction 3 s; per solve ~12 s of setup passes;
      adjoint: (4q+6d+8) s per corrector, (3q+4d+4) s for the predictor
        and assembly adjoints.
    Counts per step: 1 forward + 1 adjoint BiCGStab solve (d components
    batched), 2 correctors, the CG iterations reported."""
    s, q = 8, 2 * d + 1
    bi_it = kernel_bytes("k_bi_nm_rpv", d) + kernel_bytes("k_bi_nm_st", d) \
        if nm_bi else \
        kernel_bytes("k_bi_pv", d) + kernel_bytes("k_bi_st", d) \
        + kernel_bytes("k_bi_xr", d)
    bi_solve = s * (q + 5 * d + 1) + s * (q + 2 * d) \
        + (s * (q - 1 + 4 * d + 1) if nm_bi else 0)
    n_corr = 2
    fwd = 16 * s + (2 * d + 2) * s + n_corr * ((q + 3 * d + 1) * s
                                                + (2 * d + 2) * s)
    adj = n_corr * (4 * q + 6 * d + 8) * s + (3 * q + 4 * d + 4) * s
    cg_it = (d + 2) * s + 6 * s + 11 * s + 3 * s   # (tiled: 2 s less)
    b = (fwd + adj + bi_it * (per_step["bi_fwd"] + per_step["bi_adj"])
         + 2 * bi_solve + cg_it * per_step["cg"] + 4 * n_corr * 12 * s / 2)
    gbs = b * n / (per_step["ms"] * 1e-3) / 1e9
    return {"bytes_per_cell": b, "achieved_gbs": gbs, "peak": peak,
            "frac": gbs / peak,
            "model": "SURVEY.md §8(d) per-op bytes x this step's counts"}


def run_c5train(args, world, rank, local, dev):
    """Config 5: one training step = 16-step unrolled fwd+adjoint of the
    64x48x64 LES sample of this rank with the CNN corrector, plus the
    gradient all-reduce.  value = all ranks' cell-steps / max device time."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2505_16992_b200 import _lib, channel, les, mesh, piso
    shape, ratio, cfl, desc = CONFIGS["c5train"]
    dom = mesh.make_channel(shape, ratio=ratio)
    state, nu, u_tau = channel.reichardt_init(dom, 180.0, perturbation=0.1,
                                              seed=rank, device=dev)
    dt = cfl * (2 * np.pi / shape[0]) / float(state.u.abs().max())
    forcing = channel.WallForcing(dom, dev)
    torch.manual_seed(0)
    # the CNN corrector computes in float32 (cuDNN, tensor cores); the PISO
    # step and its adjoint stay float64
    torch.backends.cudnn.benchmark = True
    model = les.SGSCorrector(shape, dom.box_layout()[1],
                             dtype=torch.float32).to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3)
    target = state.u[:, 0].reshape(shape).mean(dim=(0, 2)).detach()
    bc = torch.cat(list(state.bc), 0)
    cfg = piso.StepConfig(dt=dt, nu=nu, tol=args.tol)
    u0 = state.u.t().contiguous().t()
    # the paper's statistics loss (S/stats.py:567-614) against the initial
    # state's statistics, turbulent-channel weights
    from paper_2505_16992_b200 import stats as S
    sl = S.channel_slices(dom)
    ref = tuple(t.detach() for t in S.frame_profile(sl, u0))
    stats_target = (ref, S.tcf_default_weights(3), sl)

    def tstep():
        return les.train_step(dom, u0, bc, model, opt, forcing, nu, cfg,
                              UNROLL, target, stats_target=stats_target)

    for _ in range(args.warmup):
        tstep()
    lib = _lib.load()
    busy = wait_for_idle_gpu(local) if world == 1 else []
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    l0 = lib.pf_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = [tstep() for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    launches = lib.pf_launch_count() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if share_dev() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * dom.n * UNROLL * args.steps / (ms / 1e3) / 1e6
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reichardt_init seed = rank)",
            "config": {"workload": desc, "grid": list(shape),
                       "cells_per_sample": dom.n, "unroll": UNROLL,
                       "sgs_cnn_dtype": "f32 (PISO step and adjoint f64)",
                       "loss": "statistics loss (S/stats.py:567-614)",
                       "samples": world, "parallelism": f"dp{world}",
                       "tol": args.tol,
                       "l2": "working set > L2 per unrolled step chain"},
            "loss_last": losses[-1], "gpu_launches": int(launches),
            "clocks": clk}))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_leg(args):
    """Bounded CPU baseline (~10 s): the reference's compiled lane, one
    single-threaded process, CPU_SAMPLE_STEPS fwd+adjoint steps of the same
    channel recipe at 64x48x64.  The same-config C4 number (one full C4
    step on one core, ~20 min, too long for this leg) is quoted from the
    committed measurement of `bench.py --impl reference` on the GPU box's
    host (profiles/r2_reference_c4.json) when present."""
    if args.config in CASES2D:
        # C1: the full config (100 steps take ~2 s on one core); C2 / C3:
        # one step of the same recipe at 1/16 of the cells
        c1 = args.config == "c1"
        try:
            r = run_reference_sample(1, 100 if c1 else 4, args.tol,
                                     ("full",) if c1 else ("sample",),
                                     args.config)
            what = ("the full C1 config, 100 fwd+adjoint steps" if c1 else
                    f"the {args.config} recipe at 1/16 of the cells, 4 "
                    f"fwd+adjoint steps")
            return {"value": r["value"], "unit": UNIT, "cores": 1,
                    "kind": "reference",
                    "sample": (f"reference pisoflow (lane {r['lane']}): "
                               f"{what}, {r['seconds']:.1f} s, 1 process"),
                    "iterations": r["iterations"]}
        except Exception as exc:
            return {"value": None, "unit": UNIT, "cores": 1,
                    "kind": "reference", "sample": f"failed: {exc}"[:200]}
    try:
        r = run_reference_sample(1, CPU_SAMPLE_STEPS, args.tol)
        cpu = {"value": r["value"], "unit": UNIT, "cores": 1,
               "kind": "reference",
               "sample": (f"reference pisoflow (lane {r['lane']}) on channel "
                          f"{'x'.join(map(str, SAMPLE_SHAPE))} (same recipe, "
                          f"1/64 of C4 cells), {CPU_SAMPLE_STEPS} fwd+adjoint"
                          f" steps, {r['seconds']:.1f} s, 1 process"),
               "iterations": r["iterations"]}
    except Exception as exc:
        cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"failed: {exc}"[:200]}
    path = os.path.join(ROOT, "profiles", "r2_reference_c4.json")
    if args.config == "c4" and os.path.exists(path):
        try:
            rec = json.load(open(path))
            cpu["same_config_c4"] = {
                k: rec.get(k) for k in ("value", "unit", "steps",
                                        "ms_per_step", "reference_seconds",
                                        "reference_iterations")}
            cpu["same_config_c4"]["source"] = (
                "profiles/r2_reference_c4.json (bench.py --impl reference "
                "on the GPU box host, committed)")
        except (OSError, ValueError):
            pass
    return cpu


def share_dev():
    return os.environ.get("PF_BENCH_SHARE_DEVICE") == "1"


def build_workload(args, dev, rank=0, world=1):
    """The C4 workload; with world > 1 this rank's slab of it (SURVEY §8 e:
    slab decomposition of the periodic streamwise axis, ghost-plane halos
    and cross-rank reductions over NVLink peer memory).  The initial field
    and the cotangent are the single-GPU ones, restricted to the slab."""
    import numpy as np
    import torch
    from paper_2505_16992_b200 import channel, mesh, piso, slab
    if args.config in CASES2D:
        dom, nu, dt, u0 = case_2d(mesh, args.config)
        g = torch.Generator(device="cpu").manual_seed(0)
        w = torch.randn((dom.n, 2), generator=g, dtype=torch.float64).to(dev)
        state = piso.make_state(dom, u0=u0, device=dev)
        return dom, state, nu, dt, (lambda u, nu_: None), w, None
    shape, ratio, cfl, _ = CONFIGS[args.config]
    dom = mesh.make_channel(shape, ratio=ratio)
    u0, nu, u_tau = channel.reichardt_velocity(dom, 180.0, perturbation=0.1,
                                               seed=0, device=dev)
    dt = cfl * (2 * np.pi / shape[0]) / float(u0.abs().max())
    g = torch.Generator(device="cpu").manual_seed(0)
    w = torch.randn((dom.n, 3), generator=g, dtype=torch.float64).to(dev)
    if world == 1:
        state = piso.make_state(dom, u0=u0, device=dev)
        return dom, state, nu, dt, channel.WallForcing(dom, dev), w, None
    sd = slab.SlabDomain(dom, rank, world)
    comm = slab.SlabComm.distributed(sd, dev)
    state = piso.make_state(sd, u0=sd.scatter(u0), device=dev)
    wl = sd.scatter(w).contiguous()
    del u0, w
    return sd, state, nu, dt, slab.SlabWallForcing(sd, dev), wl, comm


def self_launch(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: start the N ranks
    ourselves (torch.distributed.run on 127.0.0.1), one per visible GPU, and
    fail loudly when fewer than N GPUs are visible (PF_BENCH_SHARE_DEVICE=1:
    every rank on cuda:0, a correctness run of the multi-rank path)."""
    import socket
    import torch
    n = args.gpus
    vis = torch.cuda.device_count()
    if not share_dev() and vis < n:
        raise SystemExit(f"bench.py --gpus {n}: only {vis} GPU(s) visible; "
                         f"refusing to report a {n}-GPU number")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def main():
    args = parse()
    if args.reference_worker:
        return reference_worker(args)
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.config in CASES2D:
        args.tol = CASES2D[args.config][1]

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PF_BENCH_SHARE_DEVICE=1 (correctness runs of the multi-rank path on a
    # one-GPU box): every rank on cuda:0, gloo for the host-side collectives
    share = os.environ.get("PF_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2505_16992_b200 import _lib, adjoint, piso

    if args.config == "c5train":
        return run_c5train(args, world, rank, local, dev)

    # C4 splits into slabs across the ranks (strong scaling); the other
    # configs run one replica per rank (weak scaling)
    slabbed = world > 1 and args.config in ("c4", "slab8")
    dom, state0, nu, dt, forcing, w, comm = build_workload(
        args, dev, rank if slabbed else 0, world if slabbed else 1)
    plan = dom.device_plan(dev)
    cot = adjoint.GradState(u=w, p=torch.zeros(dom.n, dtype=torch.float64,
                                               device=dev))
    ws = piso.PisoWorkspace(dom)
    stats = {"mom": 0, "p": 0, "adj": 0, "steps": 0, "bi_fwd": 0,
             "bi_adj": 0, "cg": 0}

    def fwd(state):
        cfg = piso.StepConfig(dt=dt, nu=nu, source=forcing(state.u, nu),
                              tol=args.tol)
        tape = piso.StepTape()
        new, dg = piso.piso_step(dom, state, cfg, ws, tape)
        return new, dg, tape

    def adj(tape):
        return adjoint.backward_step(dom, tape, cot, tol=args.tol)

    def count(dg, g):
        stats["mom"] += dg.momentum_iterations
        stats["p"] += dg.pressure_iterations
        stats["adj"] += g.solve_iterations
        stats["bi_fwd"] += _lockstep(dg.reports, "momentum[", dom.dim)
        stats["bi_adj"] += _lockstep(g.reports or [], "adjoint_momentum",
                                     dom.dim)
        stats["cg"] += (dg.pressure_iterations
                        + sum(r.iterations for r in (g.reports or [])
                              if r.stage.startswith("adjoint_pressure")))
        stats["steps"] += 1

    def step(state):
        new, dg, tape = fwd(state)
        g = adj(tape)
        count(dg, g)
        return new, g

    state = state0
    # the warm-up holds the previous step's gradient as the timed loop does,
    # so the caching allocator reaches its high-water mark here (a first
    # cudaMalloc inside the timed loop stalled its first steps 30-140 ms)
    grad = None
    for _ in range(args.warmup):
        state, grad = step(state)
    for k in stats:
        stats[k] = 0

    lib = _lib.load()
    busy = wait_for_idle_gpu(local) if world == 1 else []
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    l0 = lib.pf_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-step events (no synchronisation) and the host's issue times: a
    # step that stalls shows whether the device or the host held it up
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    host_t = []
    trace = os.environ.get("PF_TRACE_STEPS") == "1" and rank == 0
    if trace:  # diagnosis only: per-call events (not a bench number)
        _lib.TRACE = []
        mem0 = torch.cuda.memory_stats(dev)
    e0.record()
    t_host0 = time.perf_counter()
    for k in range(args.steps):
        state, grad = step(state)
        marks[k].record()
        host_t.append(time.perf_counter())
    e1.record()
    torch.cuda.synchronize()
    if trace:
        rows = [(nm, 1e3 * (a - t_host0), 1e3 * (b - t_host0),
                 e0.elapsed_time(x), e0.elapsed_time(y))
                for nm, a, b, x, y in _lib.TRACE]
        _lib.TRACE = None
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out",
                               f"trace_{os.getpid()}.json"), "w") as f:
            mem1 = torch.cuda.memory_stats(dev)
            json.dump({"rows": rows,
                       "steps": [e0.elapsed_time(m) for m in marks],
                       "mem": {k: [mem0.get(k), mem1.get(k)] for k in (
                           "num_device_alloc", "num_device_free",
                           "num_alloc_retries",
                           "reserved_bytes.all.current")}}, f)
    prev = e0
    step_ms = []
    for mk in marks:
        step_ms.append(prev.elapsed_time(mk))
        prev = mk
    host_ms = [1e3 * (b - a) for a, b in zip([t_host0] + host_t[:-1], host_t)]
    launches = lib.pf_launch_count() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if share_dev() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    ms_step = ms / args.steps
    cells_job = (dom.global_domain.n if slabbed else world * dom.n)
    value = cells_job * args.steps / (ms / 1e3) / 1e6
    it_per_step = {k: stats[k] / max(stats["steps"], 1)
                   for k in ("mom", "p", "adj", "bi_fwd", "bi_adj", "cg")}

    # end to end through the public API with host buffers: every step's
    # input state (velocity, pressure, boundary values) is copied in from
    # pinned host memory, and its output velocity / pressure and the
    # velocity gradient are copied out to pinned host memory.  The state
    # makes a real host round trip: step k's output goes to the host and
    # comes back as step k + 1's input.  Those copies run while step k's
    # adjoint computes, in chunks on two side streams so the device-to-host
    # and host-to-device engines overlap (the gradient drains during the
    # next forward step), as a production loop would.
    n_loc, d_loc = state.u.shape
    nU, nP = state.u.numel(), state.p.numel()

    def flat(t):
        # storage-order flat view of a field ((n, d) fields are transposed
        # views of (d, n) storage)
        st_ = t.t() if t.dim() == 2 else t
        return (st_ if st_.is_contiguous() else st_.contiguous()).reshape(-1)

    def pinned(m):
        # touched once here: on the GPU boxes (virtual machines) a page's
        # first touch faults through the hypervisor, which inside the timed
        # loop stalled first steps by up to half a second
        t = torch.empty(m, dtype=torch.float64, pin_memory=True)
        t.zero_()
        return t

    u_host = [pinned(nU) for _ in range(2)]
    p_host = [pinned(nP) for _ in range(2)]
    g_host = [pinned(nU) for _ in range(2)]
    # boundary values round-trip too (outflow faces change every step)
    bc_host = [[b.detach().cpu().contiguous().pin_memory() for b in state.bc]
               for _ in range(2)]
    u_host[0].copy_(flat(state.u))
    p_host[0].copy_(flat(state.p))
    nbc = sum(b.numel() for b in bc_host[0])
    h2d = (nU + nP + nbc) * 8
    d2h = (2 * nU + nP + nbc) * 8
    main = torch.cuda.current_stream(dev)
    s_out = torch.cuda.Stream(dev)
    s_in = torch.cuda.Stream(dev)
    # large fields move in 8 chunks so the next step's upload starts behind
    # the first chunk's download; small ones (C1, C5) in one copy each --
    # every chunk is a few host-side calls and stream events, which at a
    # few ms per step cost more than the overlap gains
    n_chunks = 8 if nU * 8 >= (64 << 20) else 1

    def bcs_in(slot):
        with torch.cuda.stream(s_in):
            bcs = [b.to(dev, non_blocking=True) for b in bc_host[slot]]
            ev = torch.cuda.Event()
            ev.record(s_in)
        return bcs, ev

    def e2e_loop(nsteps, s0, t_state, n_state):
        """nsteps end-to-end steps from host slot s0; returns the device
        time, the per-step marks and where the trajectory continues."""
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(main)
        with torch.cuda.stream(s_in):
            u_in = u_host[s0].to(dev, non_blocking=True)
            p_in = p_host[s0].to(dev, non_blocking=True)
        bc_in, ev = bcs_in(s0)
        e2e_marks = []
        for k in range(nsteps):
            main.wait_event(ev)
            for t in [u_in, p_in] + bc_in:
                t.record_stream(main)
            st = piso.FlowState(u=u_in.view(d_loc, n_loc).t(), p=p_in, bc=bc_in,
                                t=t_state, step=n_state)
            new, dg, tape = fwd(st)
            t_state, n_state = new.t, new.step
            done_f = torch.cuda.Event()
            done_f.record(main)
            slot = (s0 + k + 1) % 2
            last = k + 1 == nsteps
            u_nx = None if last else torch.empty(nU, dtype=torch.float64,
                                                 device=dev)
            p_nx = None if last else torch.empty(nP, dtype=torch.float64,
                                                 device=dev)
            s_out.wait_event(done_f)
            for src, hst, dst in ((flat(new.u), u_host[slot], u_nx),
                                  (flat(new.p), p_host[slot], p_nx)):
                src.record_stream(s_out)
                m = src.numel()
                for c in range(n_chunks):
                    a, b = m * c // n_chunks, m * (c + 1) // n_chunks
                    with torch.cuda.stream(s_out):
                        hst[a:b].copy_(src[a:b], non_blocking=True)
                        e_c = torch.cuda.Event()
                        e_c.record(s_out)
                    if dst is not None:
                        s_in.wait_event(e_c)
                        with torch.cuda.stream(s_in):
                            dst[a:b].copy_(hst[a:b], non_blocking=True)
            with torch.cuda.stream(s_out):
                for hb, nb in zip(bc_host[slot], new.bc):
                    hb.copy_(nb, non_blocking=True)
                    nb.record_stream(s_out)
                e_bc = torch.cuda.Event()
                e_bc.record(s_out)
            if not last:
                u_nx.record_stream(s_in)
                p_nx.record_stream(s_in)
                u_in, p_in = u_nx, p_nx
                s_in.wait_event(e_bc)
                bc_in, ev = bcs_in(slot)
            g = adj(tape)
            count(dg, g)
            done_a = torch.cuda.Event(enable_timing=True)
            done_a.record(main)
            e2e_marks.append(done_a)
            s_out.wait_event(done_a)
            with torch.cuda.stream(s_out):
                gf = flat(g.u)
                g_host[k % 2].copy_(gf, non_blocking=True)
            gf.record_stream(s_out)
        main.wait_stream(s_out)
        main.wait_stream(s_in)
        e3.record(main)
        torch.cuda.synchronize()
        ms_e2e = e2.elapsed_time(e3)
        e2e_step_ms, prev = [], e2
        for mk in e2e_marks:
            e2e_step_ms.append(round(prev.elapsed_time(mk), 3))
            prev = mk
        return ms_e2e, e2e_step_ms, (s0 + nsteps) % 2, t_state, n_state

    # untimed warm-up of the same loop (allocator blocks, first pinned
    # transfers), then the timed run continuing the trajectory
    s0, t_state, n_state = 0, state.t, state.step
    if args.warmup > 0:
        _, _, s0, t_state, n_state = e2e_loop(args.warmup, s0, t_state,
                                              n_state)
    e2e_stats0 = dict(stats)
    ms_e2e, e2e_step_ms, _, _, _ = e2e_loop(args.steps, s0, t_state,
                                            n_state)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cpu" if share_dev() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    # the box's pinned-copy bandwidth (context for e2e: the round trip is
    # hidden under the adjoint only while the copies outrun it)
    def copy_gbs(dst, src, reps=3):
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        ea.record(main)
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        eb.record(main)
        torch.cuda.synchronize()
        return reps * src.numel() * 8 / (ea.elapsed_time(eb) / 1e3) / 1e9

    dbuf = torch.empty(nU, dtype=torch.float64, device=dev)
    pcie = {"h2d_gbs": copy_gbs(dbuf, u_host[0]),
            "d2h_gbs": copy_gbs(u_host[1], dbuf)}
    del dbuf
    e2e_it = {k: (stats[k] - e2e_stats0[k]) / max(
        stats["steps"] - e2e_stats0["steps"], 1)
        for k in ("bi_fwd", "bi_adj", "cg")}
    e2e_value = cells_job * args.steps / (ms_e2e / 1e3) / 1e6

    per_step = {k: stats[k] / max(stats["steps"], 1)
                for k in ("bi_fwd", "bi_adj", "cg")}
    per_step["ms"] = ms_step
    roofline = measure_roofline(args, dom, plan, state, nu, dt, dev,
                                per_step)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if slabbed else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (reichardt_init seed 0, random cotangent)"
                     if args.config not in CASES2D else
                     "synthetic (rest / uniform-inflow start, random "
                     "cotangent)"),
            "config": workload_config(args),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "iterations_per_step": e2e_it,
                    "pinned_copy": pcie},
            "gpu_launches": int(launches),
            "iterations_per_step": it_per_step,
        }
        line["step_ms"] = {
            "device": [round(x, 3) for x in step_ms],
            "host_issue": [round(x, 3) for x in host_ms],
            "e2e_device": e2e_step_ms}
        if busy:
            line["other_gpu_processes"] = busy
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    rc = main()
    sys.exit(rc if isinstance(rc, int) else 0)
