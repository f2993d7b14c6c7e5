"""SASS opcode mix (warp instructions executed) per kernel of an ncu report (dev tool).
usage: ncu_opmix.py report.ncu-rep [kernel_index] [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
starts = [k for k, l in enumerate(lines) if l.startswith('"Address"')]
i = starts[which]
j = starts[which + 1] - 1 if which + 1 < len(starts) else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[i:j]))))
hdr = rows[0]; ix = {h: k for k, h in enumerate(hdr)}
ops = collections.Counter(); tot = 0
for r in rows[1:]:
    if len(r) != len(hdr): continue
    toks = r[ix["Source"]].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    n = float(r[ix["Instructions Executed"]] or 0)
    ops[op] += n; tot += n
print(f"total warp instructions {tot:.0f}")
for op, n in ops.most_common(top):
    print(f"  {op:22s} {n:12.0f} {100 * n / tot:5.1f}%")
