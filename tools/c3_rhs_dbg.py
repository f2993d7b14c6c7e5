"""c3 operator at sampled centre elements: GPU (host geometry) vs oracle
patches, per part (dev tool).  usage: c3_rhs_dbg.py [scale]"""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
from helpers import patch, patch_operator, rel
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
nb = max(2, int(round(32 * scale)))
h = nb // 2
cent = sorted({i + nb * (j + nb * l) for i in (h - 1, h) for j in (h - 1, h) for l in (h - 1, h)})
base = W.build_cartesian(nb, 3, "periodic")
prob = configs.config("c3", scale, geometry="host")
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
u = torch.from_numpy(prob.state).cuda()
st = W.StateVector(u, prob.k, 3)
pos = []
for c in cent:
    ids, loc, ci = patch(base, [c], 1)
    pos.append((ids, ci[0], patch_operator(base, ids, loc, prob.k, prob.material.c, prob.material.rho,
                                           (3, 1), g=5, mapping=configs.c3_mapping)))
def show(tag, out, fn):
    got = out[cent].cpu().numpy()
    ref = np.stack([fn(po, prob.state[ids])[ci] for ids, ci, po in pos])
    print(f"{tag:12s} rel {rel(got, ref):.3e}  |ref| {np.linalg.norm(ref):.3e}", flush=True)
for parts in ("cell", "face", "both"):
    show("K " + parts, op.apply_K(st, parts).data, lambda po, x: po.apply_K(x, parts))
show("minvK both", op.apply_minv_K(st).data, lambda po, x: po.apply_inverse_mass(po.apply_K(x)))
show("rhs", op.rhs(st).data, lambda po, x: po.rhs(x))
Ku = op.apply_K(st).data
show("Minv(K u)", op.apply_inverse_mass(W.StateVector(Ku, prob.k, 3)).data,
     lambda po, x: po.apply_inverse_mass(po.apply_K(x)))
np.savez("gpurun_out/c3_centers.npz", cent=np.array(cent), rhs=op.rhs(st).data[cent].cpu().numpy(),
         K=op.apply_K(st).data[cent].cpu().numpy(), Kc=op.apply_K(st, "cell").data[cent].cpu().numpy(),
         Kf=op.apply_K(st, "face").data[cent].cpu().numpy())
