"""Warp-stall samples per CUDA source line (sass,cuda view) for kernel #k of an
ncu report (dev tool).  usage: ncu_lines.py report.ncu-rep [k] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if len(row) > 4 and row[2] == "-":
        blocks.append((func, path, row))
funcs = []
for f, _, _ in blocks:
    if f not in funcs:
        funcs.append(f)
fn = funcs[which]
rows = [(p, r) for f, p, r in blocks if f == fn]
tot = sum(float(r[4] or 0) for _, r in rows)
print(fn, "total samples", tot)
for p, r in sorted(rows, key=lambda x: -float(x[1][4] or 0))[:top]:
    print(f"{float(r[4]) / tot:6.1%} {p.split('/')[-1]}:{r[0]:>4}  {r[1][:90]}")
