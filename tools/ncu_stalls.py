"""Per-kernel stall-reason totals and top stalled SASS lines with their reasons (dev tool).
usage: ncu_stalls.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
starts = [k for k, l in enumerate(lines) if l.startswith('"Address"')]
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0      # kernel index in the report
i = starts[which]
j = starts[which + 1] - 1 if which + 1 < len(starts) else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[i:j]))))
hdr = rows[0]; body = [r for r in rows[1:] if len(r) == len(hdr)]
cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[j]: sum(float(r[j] or 0) for r in body if len(r) > j) for j in cols}
S = sum(tot.values())
print("stall totals:", ", ".join(f"{k[6:]} {v/S:.0%}" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v / S > 0.01))
si = hdr.index("Warp Stall Sampling (All Samples)")
body.sort(key=lambda r: -float(r[si] or 0))
for r in body[:top]:
    rs = sorted(((float(r[j] or 0), hdr[j][6:]) for j in cols), reverse=True)[:3]
    print(f"{r[si]:>6} {r[0][-5:]} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{int(v)}" for v, n in rs if v))
