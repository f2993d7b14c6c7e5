import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import mesh as M, slabs
from paper_1805_03981_b200._lib import lib, check
k = 4
mesh = M.build_cartesian((8, 4, 3), 3, "periodic")
geo = M.affine_geometry(mesh, k)
rng = np.random.default_rng(11)
mat = M.Material(c=rng.uniform(0.5, 2, mesh.n_elements), rho=rng.uniform(0.5, 2, mesh.n_elements))
u0 = rng.standard_normal((mesh.n_elements, 4) + (k + 1,) * 3)
op = W.AcousticOperator(mesh, geo, mat)
u = torch.from_numpy(u0).cuda()
full = op.rhs(W.StateVector(u, k, 3)).data
E = mesh.n_elements
for (b, n) in [(0, E), (0, 10), (10, E - 10), (5, 7)]:
    o = torch.zeros_like(u)
    check(lib().wk_set_element_range(op._ctx, b, n))
    check(lib().wk_rhs(op._ctx, op._ptr(u), op._ptr(o), op.stream))
    check(lib().wk_set_element_range(op._ctx, 0, -1))
    d = (o[b:b+n] - full[b:b+n]).abs().max().item()
    outside = o[:b].abs().max().item() if b > 0 else 0.0
    print("range", b, n, "maxdiff", d, "outside-written", outside, flush=True)
# slab rhs vs global rhs restricted
parts = [slabs.partition(mesh, r, 2) for r in range(2)]
sops = [slabs.SlabOperator(mesh, geo, mat, p) for p in parts]
U = [torch.from_numpy(slabs.scatter_state(u0, p)).cuda() for p in parts]
for s, x in zip(sops, U):
    s.pack(x)
for s in sops:
    p = s.part; L = p.layer
    q = sops[p.left_peer]; s.ghost[:L].copy_(q.send[q.part.n_left_export:q.part.n_left_export + L])
    q = sops[p.right_peer]; s.ghost[L:2 * L].copy_(q.send[:L])
for s, x, p in zip(sops, U, parts):
    o = torch.empty_like(x)
    check(lib().wk_rhs(s.op._ctx, s.op._ptr(x), s.op._ptr(o), s.op.stream))
    ref = full[torch.from_numpy(p.global_ids).cuda()]
    diff = (o - ref).abs().amax(dim=(1, 2, 3, 4))
    bad = torch.nonzero(diff > 0).flatten().tolist()
    print("slab", p.rank, "maxdiff", diff.max().item(), "bad elems", bad[:10], len(bad), "L", p.layer, "E", p.n_local, flush=True)
    # compare ghost vs true neighbour slices
def face_slice(u, m, s):
    idx = [slice(None)] * 5
    idx[2 + 2 - m] = -1 if s else 0
    return u[tuple(idx)].reshape(u.shape[0], 4, -1)
for s, p in zip(sops, parts):
    ul = u0[p.global_ids]
    exp = np.stack([face_slice(ul[e:e+1], f >> 1, f & 1)[0] for e, f in zip(p.export_elem, p.export_face)])
    print("send ok", p.rank, np.abs(s.send.cpu().numpy() - exp).max())
    g = s.ghost.cpu().numpy()
    errs = []
    for le, gid in enumerate(p.global_ids):
        for sd in (0, 1):
            code = p.neighbors[le, 0, sd]
            if code <= -2:
                gn = mesh.neighbors[gid, 0, sd]
                want = face_slice(u0[gn:gn+1], 0, 1 - sd)[0]
                errs.append(np.abs(g[-2 - code] - want).max())
    print("ghost ok", p.rank, max(errs), len(errs))
