"""Per-GPU kernel time of ONE rank's slab of config 5 cut into P slabs (dev
tool): the rank's stage kernels (interior + boundary launches, halo pack) on
one GPU with a no-op exchange (ghost values are irrelevant for timing).
usage: slab_rank_time.py P [steps]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_03981_b200 import configs, mesh as M, slabs
from paper_1805_03981_b200.stepping import LSRK45, compute_dt

P = int(sys.argv[1]); steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
k = 4
mesh = M.build_cartesian((128, 128, 64), 3, "periodic")
mat = configs.random_material(mesh.n_elements, seed=7)
geo = M.affine_geometry(mesh, k)
part = slabs.partition(mesh, 0, P)
class _Done:
    def wait(self):
        pass
sop = slabs.SlabOperator(mesh, geo, mat, part, exchange_fn=lambda s, g: [_Done()])
u = torch.randn((part.n_local, 4) + (k + 1,) * 3, dtype=torch.float64, device="cuda")
nxt, r = torch.empty_like(u), torch.empty_like(u)
dt = compute_dt(0.2, mesh, mat, k)
for _ in range(3):
    sop.lsrk_step(u, nxt, r, dt, LSRK45)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
cur, nx = u, nxt
for _ in range(steps):
    res = sop.lsrk_step(cur, nx, r, dt, LSRK45)
    if res is nx:
        cur, nx = nx, cur
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"P={P} rank-0 slab {part.n_local} elements: {ms:.3f} ms/LSRK step "
      f"(x{P} = {ms * P:.2f} ms vs one GPU's whole mesh)", flush=True)
