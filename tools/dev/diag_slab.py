import sys, time, threading
sys.path.insert(0, '/root/repo')
import torch
from paper_2505_16992_b200 import mesh, slab, _lib
dev = torch.device('cuda:0')
dom = mesh.make_channel((6, 4, 4), ratio=1.1)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 3
slabs = [slab.SlabDomain(dom, r, W) for r in range(W)]
comms = slab.SlabComm.local_group(slabs, dev)
glob = torch.arange(dom.n * 2, dtype=torch.float64, device=dev).reshape(2, dom.n)
fields = []
for sd in slabs:
    f = torch.full((2, sd.n), -1.0, dtype=torch.float64, device=dev)
    own = sd.owned_global_rows()
    f[:, sd.owned_slice] = glob[:, torch.as_tensor(own, device=dev)]
    fields.append(f)
torch.cuda.synchronize()
t0 = time.time()
log = []
def work(r):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        plan = slabs[r].device_plan(dev)
        log.append((r, 'launch', time.time() - t0))
        slab.halo_exchange(plan, fields[r])
        log.append((r, 'launched', time.time() - t0))
        s.synchronize()
        log.append((r, 'synced', time.time() - t0))
        try:
            comms[r].status(); log.append((r, 'status ok', 0))
        except Exception as e:
            log.append((r, 'status ERR ' + str(e)[:80], 0))
ts = [threading.Thread(target=work, args=(r,)) for r in range(W)]
for t in ts: t.start()
for t in ts: t.join()
for l in log: print(l)
for sd, f in zip(slabs, fields):
    rows = torch.as_tensor(sd._global_rows(), device=dev)
    print(sd.rank, torch.equal(f, glob[:, rows]), f[0, :16].tolist(), glob[0, rows][:16].tolist())
# sequential single-thread: launch all on separate streams from one thread
fields2 = [torch.where(f < 0, f, f) for f in fields]
