"""Dev tool: ms/step of a BASELINE config on the GPU with a device-random
state (no host state build), CUDA-graph replay, median of 3.
usage: python tools/step_time.py c5 lsrk45 [steps] [c4 ader_hdg ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_03981_b200 as W  # noqa: E402
from paper_1805_03981_b200 import configs  # noqa: E402

args = sys.argv[1:]
steps = 20
pairs = []
while args:
    cfg, scheme = args[0], args[1]
    args = args[2:]
    pairs.append((cfg, scheme))
cache = {}
for cfg, scheme in pairs:
    if cfg not in cache:
        cache.clear()
        torch.cuda.empty_cache()
        prob = configs.config(cfg, geometry="device", state=False)
        op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
        cache[cfg] = (prob, op)
    prob, op = cache[cfg]
    shape = (prob.mesh.n_elements, prob.mesh.d + 1) + (prob.k + 1,) * prob.mesh.d
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    cr = prob.schemes.get(scheme, (0.1, 1))[0]
    dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
    st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
    st.run(u, dt, 6)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        st.run(u, dt, steps)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / steps)
    print(f"{cfg} {scheme} order={op.tile_order} ms/step {statistics.median(ts):.4f} "
          f"({' '.join(f'{t:.4f}' for t in ts)})", flush=True)
    del u, st
