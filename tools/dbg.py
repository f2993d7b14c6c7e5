import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
cfg, scheme, scale = sys.argv[1], sys.argv[2], float(sys.argv[3])
prob = configs.config(cfg, scale=scale)
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
u = torch.from_numpy(prob.state).cuda()
r = st.run(u, 1e-4, int(sys.argv[4]) if len(sys.argv) > 4 else 2)
torch.cuda.synchronize()
print(cfg, scheme, scale, "ok", float(r.abs().max()))
