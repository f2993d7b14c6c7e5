"""Does the memory system itself slow down under sustained load?  Alternates
20 LSRK45 steps at config 5 with a plain device copy and prints, per round,
the step time, the copy bandwidth, SM / memory clocks, power, GPU and HBM
temperature and the throttle reasons (dev tool)."""
import subprocess, sys
sys.path.insert(0, ".")
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
def smi():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active",
                           "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout.strip()
prob = configs.config("c5")
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
st = W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)
u = torch.from_numpy(prob.state).cuda()
a = torch.empty(1 << 29, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
st.run(u, 1e-4, 6); torch.cuda.synchronize()
for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    e0, e1, e2 = (torch.cuda.Event(True) for _ in range(3))
    e0.record(); st.run(u, 1e-4, 20); e1.record()
    for _ in range(10): b.copy_(a)
    e2.record(); torch.cuda.synchronize()
    print(f"round {rnd}: step {e0.elapsed_time(e1)/20:.2f} ms  copy {10*2*a.numel()*8/e1.elapsed_time(e2)/1e6:.0f} GB/s  smi[{smi()}]", flush=True)
