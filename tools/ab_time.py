"""A/B timing: run quick LSRK/ADER timings with the package found first on PYTHONPATH (dev tool)."""
import sys, os
sys.path.insert(0, os.environ.get("WK_AB_ROOT", "."))
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
tag = os.environ.get("WK_AB_TAG", "cur")
plan = [(c.split(":")[0], c.split(":")[1], int(c.split(":")[2])) for c in sys.argv[1:]] or \
    [("c2", "lsrk45", 50), ("c5", "lsrk45", 10), ("c4", "lsrk45", 10)]
for cfg, scheme, steps in plan:
    prob = configs.config(cfg)
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
    u = torch.from_numpy(prob.state).cuda()
    st.run(u, 1e-4, 6)
    torch.cuda.synchronize()
    best = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); st.run(u, 1e-4, steps); e1.record(); torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / steps)
    ms = sorted(best)[1]
    print(f"[{tag}] {cfg} {scheme}: median {ms:.3f} ms/step (reps {', '.join(f'{b:.3f}' for b in best)})  "
          f"{prob.dofs/ms/1e6:.2f} GDoF/s  file={W.__file__[-40:]}", flush=True)
    del op, st, u
    torch.cuda.empty_cache()
