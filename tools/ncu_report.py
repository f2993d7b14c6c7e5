"""Summarise an ncu report per launch: key raw metrics, SASS opcode mix, stall
reasons and the top stall sites (dev tool; its output goes under profiles/).

usage: python tools/ncu_report.py report.ncu-rep [top_sites]

The source page lists each launch's SASS in its own section, headed by a
``"Kernel Name"`` row (each launch may repeat its section); sections are
matched to launches in order, one per distinct (kernel, launch) pair, so two
different kernels never share a table."""
import collections
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "sm__cycles_elapsed.avg.per_second"]
STALL_PREFIX = "smsp__pcsamp_warps_issue_stalled_"


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_rows(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def source_sections(rep):
    text = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    sections, cur = [], None
    for line in text.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"name": next(csv.reader([line]))[1], "lines": []}
            sections.append(cur)
        elif cur is not None:
            cur["lines"].append(line)
    return sections


def main():
    rep = sys.argv[1]
    top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    launches = raw_rows(rep)
    sections = source_sections(rep)
    # one source section per launch (ncu may print each launch's twice)
    per_launch = sections
    if len(launches) and len(sections) == 2 * len(launches):
        per_launch = sections[0::2]
    for li, (hdr, units, r) in enumerate(launches):
        name = r[hdr.index("Kernel Name")]
        print(f"=== launch {li}: {name}")
        for w in RAW:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:62s} {r[i]} {units[i]}")
        stalls = {h[len(STALL_PREFIX):]: float(r[i] or 0) for i, h in enumerate(hdr)
                  if h.startswith(STALL_PREFIX) and not h.endswith("_not_issued")
                  and r[i] not in ("", "n/a")}
        tot = sum(stalls.values())
        if tot:
            print("  stall reasons (pc samples): " + ", ".join(
                f"{k.replace('.sum', '')} {100 * v / tot:.0f}%"
                for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v / tot >= 0.01))
        if li >= len(per_launch):
            continue
        rows = list(csv.reader(io.StringIO("\n".join(per_launch[li]["lines"]))))
        h = rows[0]
        ix = {k: i for i, k in enumerate(h)}
        ops, st, total, top = collections.Counter(), collections.Counter(), 0.0, []
        for row in rows[1:]:
            if len(row) != len(h):
                continue
            toks = row[ix["Source"]].split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
            n = float(row[ix["Instructions Executed"]] or 0)
            s = float(row[ix["Warp Stall Sampling (All Samples)"]] or 0)
            ops[op] += n
            st[op] += s
            total += n
            top.append((s, row[ix["Source"]].strip()[:90]))
        print(f"  warp instructions {total:.0f}; opcode mix (share, stall samples):")
        for op, n in ops.most_common(14):
            print(f"    {op:10s} {100 * n / total:5.1f}%  {st[op]:8.0f}")
        top.sort(reverse=True)
        print("  top stall sites:")
        for s, src in top[:top_n]:
            print(f"    {s:7.0f}  {src}")


if __name__ == "__main__":
    main()
