"""Per-GPU kernel time of ONE rank's slab cut into P slabs (dev tool): the
rank's LSRK45 stage kernels (interior + boundary launches, halo pack) on one
GPU with a no-op exchange (ghost values are irrelevant for timing).
usage: slab_rank_time.py MESH P ORDER [steps]
  MESH = c5 (128x128x64, random material) or weak (32P x 32 x 32, uniform)
  ORDER = xslow | xfast (slabs._local_order)"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_03981_b200 import configs, mesh as M, slabs
from paper_1805_03981_b200.stepping import LSRK45, compute_dt

which, P, order = sys.argv[1], int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
overlap = (sys.argv[5] if len(sys.argv) > 5 else "1") == "1"
k = 4
if which == "c5":
    mesh = M.build_cartesian((128, 128, 64), 3, "periodic")
    mat = configs.random_material(mesh.n_elements, seed=7)
else:
    mesh = M.build_cartesian((32 * P, 32, 32), 3, "periodic")
    mat = M.Material.uniform(mesh)
geo = M.affine_geometry(mesh, k)
part = slabs.partition(mesh, 0, P, order=order)
class _Done:
    def wait(self):
        pass
sop = slabs.SlabOperator(mesh, geo, mat, part, exchange_fn=lambda s, g: [_Done()],
                        overlap=overlap)
u = torch.randn((part.n_local, 4) + (k + 1,) * 3, dtype=torch.float64, device="cuda")
nxt, r = torch.empty_like(u), torch.empty_like(u)
dt = compute_dt(0.2, mesh, mat, k)
for _ in range(3):
    sop.lsrk_step(u, nxt, r, dt, LSRK45)
torch.cuda.synchronize()
import time
res, host = [], []
for rep in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    h0 = time.perf_counter()
    cur, nx = u, nxt
    for _ in range(steps):
        out = sop.lsrk_step(cur, nx, r, dt, LSRK45)
        if out is nx:
            cur, nx = nx, cur
    e1.record()
    host.append((time.perf_counter() - h0) * 1e3 / steps)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / steps)
ms = sorted(res)[1]
print(f"{which} P={P} {order} overlap={int(overlap)}: rank-0 slab {part.n_local} elements: {ms:.3f} ms/LSRK step "
      f"(reps {', '.join(f'{x:.3f}' for x in res)}; host issue {min(host):.3f} ms/step)", flush=True)
