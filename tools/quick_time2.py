"""Timing of configs c3 (curved ADER-HDG) and c5 (LSRK45 + ADER-HDG) (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
jobs = [(c, s) for c, s in (a.split(":") for a in sys.argv[1:])] or [("c3", "ader_hdg"), ("c5", "lsrk45"), ("c5", "ader_hdg")]
cache = {}
for cfg, scheme in jobs:
    t0 = time.time()
    if cfg not in cache:
        prob = configs.config(cfg)
        op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
        cache[cfg] = (prob, op)
    prob, op = cache[cfg]
    st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
    u = torch.from_numpy(prob.state).cuda()
    setup = time.time() - t0
    dt = W.compute_dt(prob.schemes.get(scheme, (0.1, 1))[0], prob.mesh, prob.material, prob.k)
    st.run(u.clone(), dt, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    steps = 5
    e0.record(); out = st.run(u, dt, steps); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{cfg} {scheme}: {ms:.3f} ms/step  {prob.dofs/ms/1e6:.2f} GDoF/s  setup {setup:.1f}s  "
          f"finite={bool(torch.isfinite(out).all())} max={float(out.abs().max()):.3e}", flush=True)
