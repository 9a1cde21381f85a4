import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import ref_live as RL
R = RL.reference(); RM, RP, RA = R["mesh"], R["piso"], R["adjoint"]
from paper_2505_16992_b200 import mesh, piso, adjoint, _lib
dev = torch.device("cuda:0")
T = lambda x: torch.as_tensor(np.asarray(x, dtype=np.float64), device=dev)
for name, build in [("cav", lambda M: M.make_cavity((4, 5))), ("pois", lambda M: M.make_poiseuille((5, 4), distort=0.35))]:
    rd, d = build(RM), build(mesh)
    rng = np.random.default_rng(2)
    h = rng.standard_normal((d.n, d.dim)); bc = [rng.standard_normal((f.m, d.dim)) for f in d.bfaces]
    fl = piso.contravariant_flux(d, T(h)).cpu().numpy()
    rfl = RP.contravariant_flux(rd, h)
    print(name, "flux err", np.abs(fl - rfl).max())
    o1 = piso.divergence_rhs(d, T(h), [T(b) for b in bc]).cpu().numpy()
    o2 = piso.divergence_rhs(d, T(h), [T(b) for b in bc]).cpu().numpy()
    ref = RP.divergence_rhs(rd, h, bc)
    print(name, "div err", np.abs(o1 - ref).max(), "repeat", np.abs(o1 - o2).max())
    plan = d.device_plan(dev)
    print(name, "m", plan.m, "face_offsets", plan.face_offsets, [f.m for f in d.bfaces])
