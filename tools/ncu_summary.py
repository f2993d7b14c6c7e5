"""Summarise an ncu report: key raw metrics + SASS opcode mix + top stall sites."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
out = {}
for r in rows[2:]:
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:60s} {r[i]} {units[i]}")
            out[w] = r[i]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter(); stalls = collections.Counter(); tot = 0; top = []
    for r in rows[2:]:
        if len(r) < len(hdr): continue
        s = r[ix["Source"]].strip()
        toks = s.split()
        if not toks: continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ie = float(r[ix["Instructions Executed"]] or 0)
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op] += ie; stalls[op] += st; tot += ie
        top.append((st, s[:80]))
    print("total warp instructions", tot)
    for op, n in ops.most_common(18):
        print(f"  {op:10s} {n:12.0f} {100*n/tot:5.1f}%  stall-samples {stalls[op]:8.0f}")
    top.sort(reverse=True)
    print("top stall sites:")
    for t in top[:12]:
        print("  ", t)
