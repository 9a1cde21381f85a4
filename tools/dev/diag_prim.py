import sys, time, threading, os, ctypes
sys.path.insert(0, '/root/repo')
os.environ['PF_COMM_TIMEOUT_S'] = '2'
os.environ['CUDA_MODULE_LOADING'] = 'EAGER'
os.environ['CUDA_DEVICE_MAX_CONNECTIONS'] = '32'
os.environ['PF_MAX_BATCH'] = '4'
import torch
from paper_2505_16992_b200 import mesh, slab, _lib
dev = torch.device('cuda:0')
W = int(sys.argv[1]); MODE = sys.argv[2]; N = int(sys.argv[3])
dom = mesh.make_channel((8, 12, 8), ratio=1.1)
slabs = [slab.SlabDomain(dom, r, W) for r in range(W)]
comms = slab.SlabComm.local_group(slabs, dev)
torch.cuda.synchronize()
res = {}
bar = threading.Barrier(W)
sys.path.insert(0, '/root/repo/tests')
import test_gpu_slab as T
def work(r):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        T._prewarm(bar)
        plan = slabs[r].device_plan(dev)
        x = torch.full((plan.n,), float(r + 1), dtype=torch.float64, device=dev)
        f = torch.zeros((3, plan.n), dtype=torch.float64, device=dev)
        out = []
        for k in range(N):
            if MODE in ('red', 'mix'):
                v = ctypes.c_double()
                _lib.call('pf_reduce_sum', plan.handle, _lib.ptr(x), plan.n, _lib.ptr(plan.workspace), ctypes.byref(v), plan.stream)
                out.append(v.value)
            if MODE in ('halo', 'mix'):
                slab.halo_exchange(plan, f)
        s.synchronize()
        try:
            comms[r].status(); st = 'ok'
        except Exception as e:
            st = str(e)[:200]
        res[r] = (out[:3], out[-3:], comms[r].counters(), st)
ts = [threading.Thread(target=work, args=(r,)) for r in range(W)]
for t in ts: t.start()
for t in ts: t.join()
for r in range(W): print(r, res[r])
