import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1805_03981_b200 as W
from helpers import Case, rel
c = Case(sys.argv[1])
g = c.gpu_operator()
st = W.StateVector(torch.from_numpy(c.u).cuda(), c.k, c.d)
for var in ("ader", "ader_hdg"):
    for pol in ("none", "every_second"):
        for sh in (False, True):
            try:
                got = W.tck_evaluate(st, c.dt, g, pol, sh).data.cpu().numpy()
                print("tck", pol, sh, "%.2e" % rel(got, c.z[f"tck_{pol}_{int(sh)}"]), flush=True)
            except Exception as e:
                print("tck", pol, sh, "FAIL", str(e)[:100], flush=True); sys.exit(1)
        try:
            got = W.ader_step(st, c.dt, g, var, pol).data.cpu().numpy()
            print(var, pol, "%.2e" % rel(got, c.z[f"ader_{var}_{pol}"]), flush=True)
        except Exception as e:
            print(var, pol, "FAIL", str(e)[:100], flush=True); sys.exit(1)
