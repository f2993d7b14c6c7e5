"""Config-3 (curved) ADER-HDG timing: whole step and kernel A / kernel B
separately, CUDA events on the operator stream (dev tool).
usage: curved_time.py [scale] [steps]"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs, _lib
from paper_1805_03981_b200._lib import lib, check

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
prob = configs.config("c3", scale)
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
print(f"setup {time.time() - t0:.1f}s E={prob.mesh.n_elements}", flush=True)
st = W.make_stepper(W.SchemeConfig(scheme="ader_hdg"), op)
u = torch.from_numpy(prob.state).cuda()
dt = 1e-4
st.run(u, dt, 6)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(s); st.run(u, dt, steps); e1.record(s); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"c3 ader_hdg: {ms:.3f} ms/step  {prob.dofs / ms / 1e6:.2f} GDoF/s", flush=True)
v, y = torch.empty_like(u), torch.empty_like(u)
pol = _lib.POLICY["every_second"]
P = op._ptr
for name, fn in [("A", lambda: check(lib().wk_ader_a(op._ctx, _lib.WK_ADER_HDG, pol, P(u), P(v), P(y), dt, op.stream))),
                 ("B", lambda: check(lib().wk_ader_b(op._ctx, _lib.WK_ADER_HDG, P(u), P(v), P(y), op.stream)))]:
    for _ in range(3):
        fn()
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"kernel {name}: {e0.elapsed_time(e1) / steps:.3f} ms", flush=True)
