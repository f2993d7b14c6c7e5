import sys, ctypes, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_03981_b200 import mesh as M
from paper_1805_03981_b200._lib import lib, check, dptr, basis_table
import oracle
from paper_1805_03981_b200.configs import c3_mapping
base = oracle.build_cartesian(2, 3, "periodic")
g, k = 5, 5
nodes = torch.from_numpy(np.ascontiguousarray(M.geometry_nodes(base, g, c3_mapping))).cuda()
print("nodes", nodes.shape, nodes.dtype, nodes.is_contiguous(), flush=True)
E, d = base.n_elements, 3
gl = basis_table("gl_points", g)
pts = basis_table("gauss_points", k); w = basis_table("gauss_weights", k)
wt = np.multiply.outer(w, np.multiply.outer(w, w)).ravel()
npts = np.array([6, 6, 6], dtype=np.int32)
val = np.ascontiguousarray(np.concatenate([M.lagrange(gl, pts).ravel()] * 3))
der = np.ascontiguousarray(np.concatenate([M.lagrange(gl, pts, True).ravel()] * 3))
inv = torch.empty((E, 3, 3, 216), dtype=torch.float64, device="cuda")
jxw = torch.empty((E, 216), dtype=torch.float64, device="cuda")
for with_stats in (False, True):
    stats = torch.zeros((E, 3), dtype=torch.float64, device="cuda") if with_stats else None
    P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
    rc = lib().wk_curved_metric(d, g, E, P(nodes), dptr(npts), dptr(val), dptr(der), dptr(wt),
                                -1, 0, P(inv), P(jxw), None, P(stats), None, None)
    print("rc", rc, flush=True)
    torch.cuda.synchronize()
    print("ok stats", with_stats, float(jxw.sum()), flush=True)
