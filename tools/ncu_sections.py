"""Per-region dynamic instruction mix of each kernel in an ncu report (SASS order)."""
import csv, io, subprocess, sys
rep, E = sys.argv[1], float(sys.argv[2])
nchunks = int(sys.argv[3]) if len(sys.argv) > 3 else 16
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "?", "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for b in blocks:
    hdr = b["rows"][0]; ix = {h: i for i, h in enumerate(hdr)}
    seq = []
    for r in b["rows"][1:]:
        if len(r) < len(hdr) or r[ix["Source"]] == "Source": continue
        seq.append((r[ix["Source"]].strip(), float(r[ix["Instructions Executed"]] or 0),
                    float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    print("==", b["name"][:90])
    n = len(seq); tot = sum(c for _, c, _ in seq); step = max(1, n // nchunks)
    for k in range(0, n, step):
        chunk = seq[k:k + step]
        c = sum(x for _, x, _ in chunk); st = sum(y for _, _, y in chunk)
        if c / E < 0.5: continue
        ops = {}
        for s, x, _ in chunk:
            t = s.split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] = ops.get(op, 0) + x
        top = sorted(ops.items(), key=lambda t: -t[1])[:6]
        print(f"{k:5d}-{k + step:5d} {c / E:8.1f}/unit stall {st:6.0f}  " + " ".join(f"{o}:{v / E:.0f}" for o, v in top))
    print("total per unit", tot / E)
