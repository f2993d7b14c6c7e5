"""Build a variant of libwk_b200.so with extra nvcc flags on ONE (d, n)
instantiation, linked with the in-tree objects of all others (dev tool).
usage: variant.py NAME D N [nvcc flags...]  ->  variants/libwk_NAME.so"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as G
name, d, n, extra = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4:]
os.makedirs(os.path.join(G.ROOT, "variants"), exist_ok=True)
obj = f"/tmp/var_{name}_d{d}_n{n}.o"
subprocess.check_call([G._nvcc(), *G.NVCC_FLAGS, *extra, f"-DWK_D={d}", f"-DWK_N={n}", "-c",
                       os.path.join(G.CSRC, "wk_inst.cu"), "-o", obj])
objs = [os.path.join(G.CSRC, f) for f in sorted(os.listdir(G.CSRC))
        if f.endswith(".o") and not f.endswith("_chk.o") and f != f"wk_inst_d{d}_n{n}.o"] + [obj]
out = os.path.join(G.ROOT, "variants", f"libwk_{name}.so")
subprocess.check_call([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                       "-o", out, *objs])
print(out)
