"""Sustained timing: R repeats of K steps back to back, every repeat printed,
SM clock and board power sampled while the GPU runs (dev tool).
usage: sustain.py CONFIG SCHEME K R"""
import subprocess, sys, threading, time
sys.path.insert(0, ".")
import torch
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import configs
cfg, scheme, K, R = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
prob = configs.config(cfg)
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
st = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
u = torch.from_numpy(prob.state).cuda()
st.run(u, 1e-4, 6)
torch.cuda.synchronize()
samples, stop = [], False
def poll():
    while not stop:
        o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu",
                            "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout.strip()
        samples.append(o)
        time.sleep(0.1)
th = threading.Thread(target=poll); th.start()
out = []
for rep in range(R):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); st.run(u, 1e-4, K); e1.record(); torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1) / K)
stop = True; th.join()
import os
print(f"[{os.environ.get('WK_STREAM','dir')}] {cfg} {scheme} K={K}: " + " ".join(f"{x:.2f}" for x in out), flush=True)
print("   smi:", " | ".join(samples[::max(1, len(samples)//8)][:9]), flush=True)
