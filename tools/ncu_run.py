"""Run a few fused steps of one config/scheme eagerly, for an ncu capture
(dev tool).  usage: ncu_run.py CONFIG SCHEME [steps] [scale]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs

cfg, scheme = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
prob = configs.config(cfg, scale)
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
u = torch.from_numpy(prob.state).cuda()
st.use_graph = False
u = st.run(u, 1e-4, steps)
torch.cuda.synchronize()
print("ok", cfg, scheme, float(u.abs().max()))
