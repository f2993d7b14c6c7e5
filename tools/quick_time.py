"""Quick CUDA-event timing of the fused LSRK stage / ADER step (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
for cfg, scheme, steps in [("c2", "lsrk45", 20), ("c2", "ader_hdg", 20), ("c4", "ader_hdg", 10), ("c4", "lsrk45", 10), ("c5", "lsrk45", 10)]:
    t0 = time.time()
    prob = configs.config(cfg)
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
    u = torch.from_numpy(prob.state).cuda()
    setup = time.time() - t0
    dt = 1e-4
    st.run(u, dt, 6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); st.run(u, dt, steps); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    dofs = prob.dofs
    bpd = 160 if scheme.startswith("lsrk") else 48
    print(f"{cfg} {scheme}: {ms:.3f} ms/step  {dofs/ms/1e6:.2f} GDoF/s  HBM-equiv {bpd*dofs/ms/1e6:.0f} GB/s  setup {setup:.1f}s", flush=True)
