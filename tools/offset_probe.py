"""Is the slow state of the stage kernel a phase relation between its streams?
Runs config 5 LSRK45 with the stepper's two work vectors carved out of one
allocation at a chosen byte skew relative to a 2 MB boundary (dev tool).
usage: offset_probe.py SKEW_BYTES [K] [R]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
skew = int(sys.argv[1]); K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
R = int(sys.argv[3]) if len(sys.argv) > 3 else 6
prob = configs.config("c5")
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
st = W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)
u = torch.from_numpy(prob.state).cuda()
n = u.numel()
pool = torch.empty(2 * n + 2 * (1 << 20), dtype=torch.float64, device="cuda")
base = pool.data_ptr()
def carve(start_elems):
    return pool[start_elems:start_elems + n].view(u.shape)
a0 = (-base // 8) % (1 << 18)                 # elements up to the next 2 MB boundary
b1 = carve(a0 + skew // 8)
b2 = carve(a0 + skew // 8 + n + ((-(n)) % (1 << 18)) + 2 * (skew // 8))
st._bufs = (b1, b2)
st.run(u, 1e-4, 6); torch.cuda.synchronize()
out = []
for rep in range(R):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); st.run(u, 1e-4, K); e1.record(); torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1) / K)
print(f"skew {skew:8d} B: u%2M={u.data_ptr() % (1<<21)} b1%2M={b1.data_ptr() % (1<<21)} b2%2M={b2.data_ptr() % (1<<21)}  " + " ".join(f"{x:.2f}" for x in out), flush=True)
