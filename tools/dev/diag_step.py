import sys, time, threading, os
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
os.environ['CUDA_MODULE_LOADING'] = 'EAGER'
os.environ['CUDA_DEVICE_MAX_CONNECTIONS'] = '32'
os.environ['PF_NO_GRAPHS'] = '1'
os.environ['PF_MAX_BATCH'] = '4'
import torch
import faulthandler
faulthandler.dump_traceback_later(60, exit=True)
os.environ['PF_COMM_TIMEOUT_S'] = '1'
import test_gpu_slab as T
from paper_2505_16992_b200 import adjoint, piso, slab
W = int(sys.argv[1])
dom, dev, u0, nu, dt, w = T._setup()
t0 = time.time()
ref = T._single(dom, dev, u0, nu, dt, w, steps=1)
print('single', time.time() - t0, ref[0][1].pressure_iterations, ref[0][1].momentum_iterations, flush=True)
slabs = [slab.SlabDomain(dom, r, W) for r in range(W)]
if len(sys.argv) > 2 and sys.argv[2] == 'jacobi':
    from paper_2505_16992_b200.plan import DevicePlan
    for sd in slabs:
        sd._plans[str(dev)] = DevicePlan(sd, dev, geom_precond='multigrid')
        print('has_mg', sd._plans[str(dev)].has_mg)
comms = slab.SlabComm.local_group(slabs, dev)
torch.cuda.synchronize()
bar = threading.Barrier(W)
def work(r):
    sd = slabs[r]
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        T._prewarm(bar)
        st = piso.make_state(sd, u0=sd.scatter(u0), device=dev)
        print(r, 'state', time.time() - t0, flush=True)
        src = torch.tensor([1e-3, 0, 0], dtype=torch.float64, device=dev)
        cfg = piso.StepConfig(dt=dt, nu=nu, source=src, tol=1e-12)
        tape = piso.StepTape()
        try:
            st, diag = piso.piso_step(sd, st, cfg, None, tape)
        except Exception as e:
            print(r, 'EXC', e, flush=True)
        try:
            comms[r].status()
        except Exception as e:
            print(r, 'STATUS', e, flush=True)
            return
        print(r, 'fwd', time.time() - t0, diag.pressure_iterations, diag.momentum_iterations, flush=True)
        comms[r].status()
        g = adjoint.backward_step(sd, tape, adjoint.GradState(u=sd.scatter(w), p=torch.zeros(sd.n, dtype=torch.float64, device=dev)), tol=1e-12)
        print(r, 'bwd', time.time() - t0, g.solve_iterations, g.nu, flush=True)
        comms[r].status()
from paper_2505_16992_b200 import _lib as L
orig = L.call
tl = threading.local()
traces = {}
def traced(name, *args):
    rc = orig(name, *args)
    r = getattr(tl, 'rank', None)
    if r is not None and not name.startswith('pf_comm'):
        traces.setdefault(r, []).append((name, comms[r].counters()))
    return rc
L.call = traced
def work0(r):
    tl.rank = r
    work(r)
ts = [threading.Thread(target=work0, args=(r,)) for r in range(W)]
for t in ts: t.start()
for t in ts: t.join()
print('done', time.time() - t0)
for k in range(max(len(v) for v in traces.values())):
    row = [traces[r][k] if k < len(traces[r]) else None for r in range(W)]
    flag = '' if all(x == row[0] for x in row) else '   <<<< DIFF'
    print(k, row, flag)
