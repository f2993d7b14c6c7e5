"""Config-3 setup time: host vs device geometry (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1805_03981_b200 import configs
import paper_1805_03981_b200 as W
for geo in ("device", "host"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = configs.config("c3", geometry=geo)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    torch.cuda.synchronize()
    print(f"{geo}: config {t1 - t0:.2f} s, operator {time.perf_counter() - t1:.2f} s", flush=True)
    del op, prob
